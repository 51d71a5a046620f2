#!/bin/bash
# the round's final bench lines (no ncu): default run, sync prepare, the other configs, reference arm
mkdir -p gpurun_out/final
timeout 600 python bench.py > gpurun_out/final/bench_cfg2.json 2> gpurun_out/final/bench_cfg2.err
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
timeout 600 python bench.py --no-prefetch --no-cpu-baseline > gpurun_out/final/bench_cfg2_sync.json 2> /dev/null
timeout 600 python bench.py --config small > gpurun_out/final/bench_small.json 2> /dev/null
timeout 600 python bench.py --config avazu > gpurun_out/final/bench_avazu.json 2> /dev/null
timeout 900 python bench.py --config stress > gpurun_out/final/bench_stress.json 2> /dev/null
