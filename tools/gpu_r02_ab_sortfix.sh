# A/B: the sort-state address fix (current .so) vs the build before it (build/ab/libold.so), cfg2, alternating
mkdir -p gpurun_out/ab
for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab/new_$i.json 2>/dev/null
  FC_LIB_PATH=build/ab/libold.so timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab/old_$i.json 2>/dev/null
done
for f in gpurun_out/ab/*.json; do python -c "
import json; d=json.load(open('$f')); e=d.get('e2e') or {}
print('$f'.split('/')[-1], round(d['value']/1e6,1), round(d['ms_per_step'],3), round(e['value']/1e6,1), d['step_latency_ms']['update_avg'], d['clocks']['reasons'])"; done
