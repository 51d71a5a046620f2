#!/bin/bash
# depth 1 vs 2 on avazu and stress + the updated pipeline tests
timeout 600 python -m pytest tests/test_gpu_abi_errors.py tests/test_gpu_prefetch.py -q -x 2>&1 | tail -2
for cfg in avazu stress; do
for i in 1 2 3; do
  for d in 1 2; do
    timeout 600 python bench.py --config $cfg --prefetch-depth $d --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/d2.json 2>gpurun_out/d2.err
    python -c "import json;d=json.loads(open('gpurun_out/d2.json').read().strip().splitlines()[-1]);e=d['e2e'];print('$cfg depth $d run $i', round(d['value']/1e6,1), round(d['ms_per_step'],4), 'e2e', round(e['value']/1e6,1), 'p50/p99', d['step_latency_ms']['p50'], d['step_latency_ms']['p99'])"
  done
done
done
