mkdir -p gpurun_out
rm -f gpurun_out/fused.txt
timeout 300 python -m pytest tests/test_gpu_prefetch.py -q -x > gpurun_out/pytest_pf.log 2>&1; echo rc=$? >> gpurun_out/pytest_pf.log
for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_v.json 2> /dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_v.json')); print(round(d['value']/1e6,1), round(d['ms_per_step'],3), round(d['e2e']['value']/1e6,1), d['step_latency_ms']['update_avg'])" >> gpurun_out/fused.txt
done
