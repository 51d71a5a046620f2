# FC_TMA_BLOCKS re-sweep of the pipelined staging on the closing build, cfg2, alternating
mkdir -p gpurun_out/tma; rm -f gpurun_out/tma/*.json
for i in 1 2 3; do
  for b in ${BLOCKS:-32 40 48 56}; do
    FC_TMA_BLOCKS=$b timeout 600 python bench.py --no-cpu-baseline > gpurun_out/tma/b${b}_$i.json 2>/dev/null
  done
done
for f in gpurun_out/tma/*.json; do python -c "
import json; d=json.load(open('$f')); e=d.get('e2e') or {}
print('$f'.split('/')[-1], round(d['value']/1e6,1), round(d['ms_per_step'],3), round(e['value']/1e6,1), round(d['step_latency_ms']['miss_transfer_avg'],3), round(d['step_latency_ms']['update_avg'],3))"; done
