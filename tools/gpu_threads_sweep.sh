#!/bin/bash
# host scatter threads (FC_SCATTER_THREADS) on cfg2 and stress, alternating
for cfg in criteo_kaggle stress; do
for i in 1 2; do
  for t in 4 8 12; do
    FC_SCATTER_THREADS=$t timeout 600 python bench.py --config $cfg --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/th.json 2>gpurun_out/th.err
    python -c "import json;d=json.loads(open('gpurun_out/th.json').read().strip().splitlines()[-1]);e=d['e2e'];sl=d['step_latency_ms'];print('$cfg threads $t run $i', round(d['value']/1e6,1), round(d['ms_per_step'],4), 'e2e', round(e['value']/1e6,1), 'p99', round(sl['p99'],3), 'scatter', round(sl['host_scatter_avg'],3))"
  done
done
done
