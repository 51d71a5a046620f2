# Which chain bounds the pipelined cfg2 step: k empty kernels appended to every index phase
# (FC_DEBUG_NOOP_INDEX) or put before every staging (FC_DEBUG_NOOP_XFER), alternating on one box
mkdir -p gpurun_out/noopc
for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/noopc/base_$i.json 2>/dev/null
  for k in 2 4; do
    FC_DEBUG_NOOP_INDEX=$k timeout 600 python bench.py --no-cpu-baseline > gpurun_out/noopc/index${k}_$i.json 2>/dev/null
    FC_DEBUG_NOOP_XFER=$k timeout 600 python bench.py --no-cpu-baseline > gpurun_out/noopc/xfer${k}_$i.json 2>/dev/null
  done
done
for f in gpurun_out/noopc/*.json; do python -c "
import json; d=json.load(open('$f')); e=d.get('e2e') or {}
print('$f'.split('/')[-1], round(d['value']/1e6,1), round(d['ms_per_step'],3), round(e['value']/1e6,1), round(d['step_latency_ms']['update_avg'],3), round(d['step_latency_ms']['miss_transfer_avg'],3))"; done
