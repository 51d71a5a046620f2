mkdir -p gpurun_out/final
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.log
timeout 600 python bench.py > gpurun_out/final/bench_cfg2.json 2> gpurun_out/final/bench_cfg2.err
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
timeout 600 python bench.py --no-prefetch --no-cpu-baseline > gpurun_out/final/bench_cfg2_sync.json 2> /dev/null
timeout 600 python bench.py --config small > gpurun_out/final/bench_small.json 2> /dev/null
timeout 600 python bench.py --config avazu > gpurun_out/final/bench_avazu.json 2> /dev/null
timeout 900 python bench.py --config stress > gpurun_out/final/bench_stress.json 2> /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for k in k_admit_stage_tma k_pool1 k_bwd_stream k_bits_emit k_mark_ids k_evict_commit k_admit_commit; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 8 -c 1 \
     -o gpurun_out/final/full_${k} -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
