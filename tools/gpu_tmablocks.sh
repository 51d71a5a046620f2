mkdir -p gpurun_out
rm -f gpurun_out/tmablocks.txt
for b in 16 32 48 64 96 148; do
  FC_TMA_BLOCKS=$b timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_v.json 2> /dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_v.json')); print('$b', round(d['value']/1e6,1), round(d['ms_per_step'],3), round(d['e2e']['value']/1e6,1), {k:round(v,3) for k,v in d['step_latency_ms'].items() if v})" >> gpurun_out/tmablocks.txt
done
