mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 600 python bench.py --no-prefetch --no-cpu-baseline > gpurun_out/bench_cfg2_nopf.json 2> gpurun_out/bench_cfg2_nopf.err
timeout 600 python bench.py --config avazu > gpurun_out/bench_avazu.json 2> gpurun_out/bench_avazu.err
timeout 900 python bench.py --config stress > gpurun_out/bench_stress.json 2> gpurun_out/bench_stress.err
timeout 600 python bench.py --config small > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err
