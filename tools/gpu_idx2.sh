mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches_idx2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
rm -f gpurun_out/idx2.txt
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_v.json 2> /dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_v.json')); print(round(d['value']/1e6,1), round(d['ms_per_step'],3), round(d['e2e']['value']/1e6,1), d['gpu_launches'])" >> gpurun_out/idx2.txt
done
