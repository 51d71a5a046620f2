#!/bin/bash
mkdir -p gpurun_out
FC_TORCH_TRACE=gpurun_out/trace_sharded.json timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --sharded --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/bench_sharded_t.json 2> gpurun_out/bench_sharded_t.err
echo "sharded rc=$?"
FC_TORCH_TRACE=gpurun_out/trace_single.json timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/bench_single_t.json 2> gpurun_out/bench_single_t.err
echo "single rc=$?"
python tools/trace_gaps.py gpurun_out/trace_sharded.json > gpurun_out/gaps_sharded.txt 2>&1
python tools/trace_gaps.py gpurun_out/trace_single.json > gpurun_out/gaps_single.txt 2>&1
gzip -f gpurun_out/trace_sharded.json gpurun_out/trace_single.json
