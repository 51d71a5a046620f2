#!/bin/bash
# prefetch depth 2: parity tests, then depth 1 vs 2 on the three single-GPU configs (alternating)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prefetch.py tests/test_gpu_fullsize.py tests/test_gpu_simulator.py tests/test_gpu_embedding.py -x -q > gpurun_out/depth2_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/depth2_tests.log
for cfg in criteo_kaggle avazu stress; do
  for i in 1 2; do
    for d in 1 2; do
      timeout 600 python bench.py --config $cfg --prefetch-depth $d --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/d2.json 2>gpurun_out/d2.err
      python -c "import json;d=json.loads(open('gpurun_out/d2.json').read().strip().splitlines()[-1]);print('$cfg depth $d run $i', round(d['value']/1e6,1), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']/1e6,1))" || tail -3 gpurun_out/d2.err
    done
  done
done
