#!/bin/bash
mkdir -p gpurun_out
FC_TORCH_TRACE=gpurun_out/trace_row2048.json timeout 600 python bench.py --shard row --batch 2048 --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/tr_row.json 2>gpurun_out/tr_row.err
FC_TORCH_TRACE=gpurun_out/trace_single2048.json timeout 600 python bench.py --batch 2048 --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/tr_single.json 2>gpurun_out/tr_single.err
python tools/trace_steps.py gpurun_out/trace_row2048.json > gpurun_out/steps_row2048.txt
python tools/trace_steps.py gpurun_out/trace_single2048.json > gpurun_out/steps_single2048.txt
python tools/trace_gaps.py gpurun_out/trace_row2048.json > gpurun_out/gaps_row2048.txt
gzip -f gpurun_out/trace_row2048.json gpurun_out/trace_single2048.json
tail -3 gpurun_out/tr_row.err
