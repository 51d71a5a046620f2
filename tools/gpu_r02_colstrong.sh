#!/bin/bash
# One rank's share of the column-wise split at N = 2/4/8 (cfg2 global batch, D/N columns), timed at
# world 1: the per-rank compute + host-link work without the NCCL exchanges.
mkdir -p gpurun_out
for d in 64 32 16; do
  timeout 600 python bench.py --shard column --dim $d --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/colstrong_$d.json 2>gpurun_out/colstrong_$d.err
  timeout 600 python bench.py --dim $d --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/single_dim_$d.json 2>/dev/null
done
for f in gpurun_out/colstrong_*.json gpurun_out/single_dim_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']/1e6,1), round(d['ms_per_step'],3), round(d['e2e']['value']/1e6,1), round(d['e2e']['host_step_ms']['p50'],3), d['step_latency_ms'].get('miss_transfer_avg'))" 2>&1 | tail -1; done
tail -3 gpurun_out/colstrong_16.err
