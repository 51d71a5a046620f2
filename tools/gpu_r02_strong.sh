#!/bin/bash
# Strong-scaling floor at one GPU: the row-sharded step at the per-rank batch of N = 1/2/4/8
# (global batch 16384 split N ways), and the unsharded module at the same batches.
mkdir -p gpurun_out
for b in 16384 8192 4096 2048; do
  timeout 600 python bench.py --shard row --batch $b --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/strong_row_$b.json 2> gpurun_out/strong_row_$b.err
  timeout 600 python bench.py --batch $b --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/strong_single_$b.json 2> gpurun_out/strong_single_$b.err
done
for f in gpurun_out/strong_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']/1e6,1), round(d['ms_per_step'],3), round(d['e2e']['value']/1e6,1), d['e2e']['host_step_ms']['p50'], d['step_latency_ms'])"; done
