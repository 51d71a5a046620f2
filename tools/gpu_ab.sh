#!/bin/bash
# A/B of an env toggle on the headline bench, alternating, same box: gpu_ab.sh VAR
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in 0 1; do
    if [ $v = 1 ]; then export $1=1; else unset $1; fi
    timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${v}_$i.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/ab_${v}_$i.json').read().strip().splitlines()[-1]);print('$1=$v run $i', round(d['value']/1e6,1), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']/1e6,1))"
  done
done
