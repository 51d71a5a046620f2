#!/bin/bash
# depth 1 vs 2 on the headline config, 4 alternating rounds
for i in 1 2 3 4; do
  for d in 1 2; do
    timeout 600 python bench.py --prefetch-depth $d --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/d2.json 2>gpurun_out/d2.err
    python -c "import json;d=json.loads(open('gpurun_out/d2.json').read().strip().splitlines()[-1]);e=d['e2e'];print('depth $d run $i', round(d['value']/1e6,1), round(d['ms_per_step'],4), 'e2e', round(e['value']/1e6,1), 'host p50', round(e['host_step_ms']['p50'],3))"
  done
done
