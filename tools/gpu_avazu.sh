mkdir -p gpurun_out
rm -f gpurun_out/avazu_var.txt
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for c in avazu avazu criteo_kaggle criteo_kaggle; do
timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_v.json 2> /dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_v.json')); print('$c', round(d['value']/1e6,1), round(d['ms_per_step'],3), round(d['e2e']['value']/1e6,1), round(d['e2e']['ms_per_step'],3), d['e2e']['host_step_ms'])" >> gpurun_out/avazu_var.txt
done
