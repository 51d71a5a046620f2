mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_cache.py tests/test_gpu_embedding.py -x -q > gpurun_out/pytest_tma2.log 2>&1; echo rc=$? >> gpurun_out/pytest_tma2.log
timeout 600 python bench.py --no-cpu-baseline --no-prefetch > gpurun_out/bench_sync.json 2> gpurun_out/bench_sync.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_pf.json 2> gpurun_out/bench_pf.err
