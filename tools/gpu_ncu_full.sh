mkdir -p gpurun_out
for k in k_admit_stage_tma k_admit_commit k_evict_commit k_pool1 k_bwd_stream k_os_scatter; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 6 -c 1 \
     -o gpurun_out/full_${k} -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_${k}.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_admit_async_tma" -s 6 -c 1 \
     -o gpurun_out/full_k_admit_async_tma -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-prefetch > gpurun_out/ncu_full_async_tma.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_pf.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_pf.log 2>&1
