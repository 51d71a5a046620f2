# bounded staging: memory tests, the full GPU suite, default bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_memory.py -x -q -s 2>&1 | grep -E "passed|failed|MemGetInfo|Error|assert" | tail -15 > gpurun_out/mem_tests.txt
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gpu_tests.txt
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
