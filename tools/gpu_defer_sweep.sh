#!/bin/bash
# deferred staging (FC_XFER_AFTER_UPDATE=1) at several staging grids vs the default overlap
for i in 1 2; do
  for cfg in "default" "defer:40" "defer:64" "defer:148"; do
    unset FC_XFER_AFTER_UPDATE FC_TMA_BLOCKS
    if [ "$cfg" != default ]; then export FC_XFER_AFTER_UPDATE=1 FC_TMA_BLOCKS=${cfg#defer:}; fi
    timeout 600 python bench.py ${BENCH_ARGS:-} --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/ds.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/ds.json').read().strip().splitlines()[-1]);print('$cfg run $i', round(d['value']/1e6,1), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']/1e6,1))"
  done
done
