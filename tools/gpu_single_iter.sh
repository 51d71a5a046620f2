#!/bin/bash
# single-GPU pipelined step: bench x2 + a CUPTI gap/kernel report
mkdir -p gpurun_out
for i in 1 2; do
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_single_$i.json 2> gpurun_out/bench_single_$i.err
  echo "bench $i rc=$?"
done
FC_TORCH_TRACE=gpurun_out/trace_single.json timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
python tools/trace_gaps.py gpurun_out/trace_single.json > gpurun_out/gaps_single.txt 2>&1
gzip -f gpurun_out/trace_single.json
