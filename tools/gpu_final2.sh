#!/bin/bash
# end-of-round refresh: full GPU suite, smoke, bench lines, launch list + ncu captures of the current code
mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/final/pytest_gpu.log
bash tools/gpu_final.sh
