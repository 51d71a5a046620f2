#!/bin/bash
# sweep an env knob on the headline bench, two rounds, same box: gpu_sweep.sh VAR v1 v2 ...
mkdir -p gpurun_out
var=$1; shift
for i in 1 2; do
  for v in "$@"; do
    if [ "$v" = "-" ]; then unset $var; else export $var=$v; fi
    timeout 600 python bench.py ${BENCH_ARGS:-} --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/sw_${v}_$i.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/sw_${v}_$i.json').read().strip().splitlines()[-1]);print('$var=$v run $i', round(d['value']/1e6,1), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']/1e6,1))"
  done
done
