#!/bin/bash
mkdir -p gpurun_out
FC_TORCH_TRACE=gpurun_out/trace_col16.json FC_TORCH_TRACE_E2E=gpurun_out/trace_col16_e2e.json timeout 600 python bench.py --shard column --dim 16 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/tr_col16.json 2>gpurun_out/tr_col16.err
python tools/trace_steps.py gpurun_out/trace_col16.json > gpurun_out/steps_col16.txt
python tools/trace_steps.py gpurun_out/trace_col16_e2e.json > gpurun_out/steps_col16_e2e.txt
python tools/trace_gaps.py gpurun_out/trace_col16.json > gpurun_out/gaps_col16.txt
python tools/trace_gaps.py gpurun_out/trace_col16_e2e.json > gpurun_out/gaps_col16_e2e.txt
gzip -f gpurun_out/trace_col16*.json
head -3 gpurun_out/gaps_col16.txt gpurun_out/gaps_col16_e2e.txt
