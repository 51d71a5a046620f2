mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_router.py -x -q > gpurun_out/pytest_router.log 2>&1; echo rc=$? >> gpurun_out/pytest_router.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --sharded --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sharded.json 2> gpurun_out/bench_sharded.err
