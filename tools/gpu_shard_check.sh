#!/bin/bash
# row-sharded path: GPU tests, world-1 bench (peer + NCCL return), launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_router.py tests/test_gpu_peer.py tests/test_gpu_embedding.py -x -q > gpurun_out/shard_tests.log 2>&1
echo "tests rc=$?"
tail -3 gpurun_out/shard_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29521 bench.py --sharded --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_sharded.json 2> gpurun_out/bench_sharded.err
echo "bench rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29522 bench.py --sharded --no-peer --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_sharded_nopeer.json 2> gpurun_out/bench_sharded_nopeer.err
echo "bench nopeer rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_sharded2.csv python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29523 bench.py --sharded --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo "ncu rc=$?"
