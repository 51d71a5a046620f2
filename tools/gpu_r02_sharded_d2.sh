#!/bin/bash
# Row-sharded module with two batches in flight: GPU tests, then depth 1 vs 2 at the
# strong-scaling per-rank batches (world 1), alternating.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_router.py tests/test_gpu_column.py -x -q 2>&1 | tail -3 > gpurun_out/d2_tests.log
for rep in 1 2; do
for b in 2048 16384; do
  for d in 1 2; do
    timeout 600 python bench.py --shard row --batch $b --prefetch-depth $d --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/d2_row_${b}_d${d}_$rep.json 2>/dev/null
  done
done
done
timeout 600 python bench.py --shard column --prefetch-depth 2 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/d2_col_16384_d2.json 2>/dev/null
timeout 600 python bench.py --shard column --prefetch-depth 1 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/d2_col_16384_d1.json 2>/dev/null
cat gpurun_out/d2_tests.log
for f in gpurun_out/d2_*.json; do python -c "
import json,sys; d=json.load(open('$f')); print('$f', round(d['value']/1e6,1), round(d['ms_per_step'],3), round(d['e2e']['value']/1e6,1), round(d['e2e']['host_step_ms']['p50'],3))" 2>&1 | tail -1; done
