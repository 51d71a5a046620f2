mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_prefetch.py -q -x > gpurun_out/pytest_emb.log 2>&1; echo rc=$? >> gpurun_out/pytest_emb.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bwd.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
