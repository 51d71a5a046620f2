mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_prefetch.py -x -q > gpurun_out/pytest_prefetch.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_prefetch.log
FC_XFER_AFTER_UPDATE=1 timeout 300 python -m pytest tests/test_gpu_prefetch.py -x -q > gpurun_out/pytest_prefetch_defer.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_prefetch_defer.log
for d in 0 1; do FC_XFER_AFTER_UPDATE=$d timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_d$d.json 2> gpurun_out/bench_d$d.err; done
FC_XFER_AFTER_UPDATE=1 timeout 600 python bench.py --no-cpu-baseline --config avazu > gpurun_out/bench_avazu_d1.json 2> gpurun_out/bench_avazu_d1.err
FC_XFER_AFTER_UPDATE=1 timeout 600 python bench.py --no-cpu-baseline --config stress > gpurun_out/bench_stress_d1.json 2> gpurun_out/bench_stress_d1.err
