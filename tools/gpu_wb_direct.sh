#!/bin/bash
# (historical record: FC_WB_DIRECT / k_wb_direct were removed after this sweep; see profiles/r01_wb_direct_sweep.txt)
# direct write-back (FC_WB_DIRECT=1): parity tests, then A/B vs host scatter and a grid sweep
FC_WB_DIRECT=1 timeout 900 python -m pytest tests/test_gpu_prefetch.py tests/test_gpu_fullsize.py tests/test_gpu_embedding.py tests/test_gpu_simulator.py -x -q 2>&1 | tail -2
for i in 1 2; do
  for v in 0 16 32 64 148; do
    if [ $v = 0 ]; then unset FC_WB_DIRECT FC_WB_DIRECT_BLOCKS; else export FC_WB_DIRECT=1 FC_WB_DIRECT_BLOCKS=$v; fi
    timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/wd.json 2>gpurun_out/wd.err
    python -c "import json;d=json.loads(open('gpurun_out/wd.json').read().strip().splitlines()[-1]);e=d['e2e'];print('direct blocks $v run $i', round(d['value']/1e6,1), round(d['ms_per_step'],4), 'e2e', round(e['value']/1e6,1))" || tail -3 gpurun_out/wd.err
  done
done
