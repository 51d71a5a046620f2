mkdir -p gpurun_out
rm -f gpurun_out/e2e_dbg.txt
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for i in 1 2 3 4; do
  FC_DEBUG_WAITS=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_v.json 2> gpurun_out/bench_v.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_v.json')); print(round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), d['e2e']['host_step_ms'])" >> gpurun_out/e2e_dbg.txt
  grep "slow host wait" gpurun_out/bench_v.err | head -8 >> gpurun_out/e2e_dbg.txt
done
