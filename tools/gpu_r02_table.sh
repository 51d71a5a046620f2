#!/bin/bash
# Table-wise sharding: router/module GPU tests, then bench --shard table vs row at N=1.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_router.py -x -q 2>&1 | tail -5 > gpurun_out/table_tests.log
for sh in table row; do
  timeout 600 python bench.py --shard $sh --steps 20 --warmup 5 > gpurun_out/bench_$sh.json 2> gpurun_out/bench_$sh.err
done
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 > gpurun_out/gpu_suite.log
cat gpurun_out/table_tests.log gpurun_out/bench_*.json gpurun_out/gpu_suite.log
