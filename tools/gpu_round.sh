#!/bin/bash
# One GPU session: build check, gpu tests, smoke, bench (default), launch list, ncu --set full of top kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --config small > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
for k in ${NCU_KERNELS:-k_admit_async k_pool1 k_evict_async k_bwd_stream}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 5 -c 1 \
     -o gpurun_out/full_${k} -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_${k}.log 2>&1
done
ls -la gpurun_out
