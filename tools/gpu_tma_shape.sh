#!/bin/bash
# (historical record: the FC_TMA_STAGES knob was removed after this sweep; 4 stages are compiled in)
# staging shape: stages per block x blocks (same bytes in flight along the diagonal)
for i in 1 2; do
  for sb in 4:40 2:80 8:20 2:40 8:40; do
    export FC_TMA_STAGES=${sb%:*} FC_TMA_BLOCKS=${sb#*:}
    timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/ts.json 2>gpurun_out/ts.err
    python -c "import json;d=json.loads(open('gpurun_out/ts.json').read().strip().splitlines()[-1]);print('stages:blocks $sb run $i', round(d['value']/1e6,1), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']/1e6,1), 'stage_ms', round(d['roofline']['launch_ms'],3))" || tail -2 gpurun_out/ts.err
  done
done
