mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02_q_cfg2.json 2> gpurun_out/r02_q_cfg2.err
python -m pytest tests/test_gpu_column.py tests/test_gpu_prefetch.py tests/test_gpu_cache.py -x -q 2>&1 | tail -5 > gpurun_out/r02_q_tests.txt
