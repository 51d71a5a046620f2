# Price of a kernel boundary on the compute stream inside the pipelined cfg2 step:
# k empty kernels before each backward (FC_DEBUG_NOOP_LAUNCHES), alternating on one box
mkdir -p gpurun_out/noop
for i in 1 2 3; do
  for k in 0 2 4; do
    FC_DEBUG_NOOP_LAUNCHES=$k timeout 600 python bench.py --no-cpu-baseline > gpurun_out/noop/k${k}_$i.json 2>/dev/null
  done
done
for f in gpurun_out/noop/*.json; do python -c "
import json; d=json.load(open('$f')); e=d.get('e2e') or {}
print('$f'.split('/')[-1], round(d['value']/1e6,1), round(d['ms_per_step'],3), round(e['value']/1e6,1), round(d['step_latency_ms']['update_avg'],3), round(d['step_latency_ms']['pool_avg'],3))"; done
