mkdir -p gpurun_out
for i in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_e2e_$i.json 2> gpurun_out/bench_e2e_$i.err; done
