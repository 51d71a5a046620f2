mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_embedding.py tests/test_gpu_prefetch.py -x -q > gpurun_out/pytest_fused.log 2>&1; echo rc=$? >> gpurun_out/pytest_fused.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_sort.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-prefetch > gpurun_out/ncu_bench.log 2>&1
