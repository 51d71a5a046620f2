#!/bin/bash
# row-sharded iteration: GPU tests touching the exchange + bench (peer / NCCL) + a CUPTI gap report
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_router.py tests/test_gpu_peer.py tests/test_gpu_prefetch.py tests/test_gpu_embedding.py -x -q > gpurun_out/shard_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/shard_tests.log
for v in peer nopeer; do
  extra=""; [ $v = nopeer ] && extra="--no-peer"
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2954${#v} bench.py --sharded $extra --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_sharded_$v.json 2> gpurun_out/bench_sharded_$v.err
  echo "bench $v rc=$?"
done
FC_TORCH_TRACE=gpurun_out/trace_sharded.json timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29549 bench.py --sharded --steps 10 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
python tools/trace_gaps.py gpurun_out/trace_sharded.json > gpurun_out/gaps_sharded.txt 2>&1
gzip -f gpurun_out/trace_sharded.json
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_single.json 2> gpurun_out/bench_single.err
echo "single rc=$?"
