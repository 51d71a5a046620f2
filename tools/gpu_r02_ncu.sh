# round-2 evidence: memory test, bench line, one ncu --set full capture of a pipelined step's kernels,
# the launch list of the same command
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_memory.py -x -q -s 2>&1 | grep -E "passed|failed|MemGetInfo|Error|assert" | tail -8 > gpurun_out/mem_tests.txt
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"^(k_pool1|k_bwd_stream|k_bwd_fixup|k_os_hist|k_os_scatter|k_admit_stage_tma|k_admit_commit|k_evict_commit|k_unique_info|k_mark_ids|k_inverse)" \
  -s 120 -c 14 -o gpurun_out/r02_full -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_launches_final.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
