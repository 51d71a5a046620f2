mkdir -p gpurun_out
for v in "X=1" "FC_INDEX_ON_MAIN=1" "FC_XFER_AFTER_UPDATE=1" "FC_HOST_WAIT=1" "FC_XFER_TMA=0"; do
  env $v timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_v.json 2> /dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_v.json')); print('$v', round(d['value']/1e6,1), round(d['ms_per_step'],3), round(d['e2e']['value']/1e6,1), {k:round(v,3) for k,v in d['step_latency_ms'].items() if v})" >> gpurun_out/variants.txt
done
