mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for k in ${NCU_KERNELS:-k_admit_stage k_evict_commit k_admit_commit k_pool1 k_bwd_stream k_bwd_fixup k_bwd_apply k_mark_ids k_unique_info}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 6 -c 1 \
     -o gpurun_out/full_${k} -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_${k}.log 2>&1
done
