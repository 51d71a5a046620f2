# round-2 evidence on the current build: GPU suite + smoke, every bench line, reference arm,
# launch list and one ncu --set full capture of a pipelined step's kernels
mkdir -p gpurun_out/final2
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/final2/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final2/smoke.txt 2>&1
for i in 1 2; do timeout 600 python bench.py > gpurun_out/final2/cfg2_$i.json 2> gpurun_out/final2/cfg2_$i.err; done
for c in small avazu stress; do timeout 900 python bench.py --config $c > gpurun_out/final2/$c.json 2> gpurun_out/final2/$c.err; done
timeout 600 python bench.py --gpus 1 --shard column --no-cpu-baseline > gpurun_out/final2/cfg2_col.json 2> gpurun_out/final2/cfg2_col.err
timeout 900 python bench.py --config criteo_1tb --gpus 1 --shard column --no-cpu-baseline > gpurun_out/final2/1tb_col.json 2> gpurun_out/final2/1tb_col.err
timeout 600 python bench.py --gpus 1 --shard row --no-cpu-baseline > gpurun_out/final2/cfg2_row.json 2> gpurun_out/final2/cfg2_row.err
timeout 600 python bench.py --impl reference > gpurun_out/final2/ref.json 2> gpurun_out/final2/ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final2/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"^(k_pool1|k_bwd_stream|k_bwd_fixup|k_os_scatter|k_admit_stage_tma|k_admit_commit|k_evict_commit|k_unique_info|k_mark_ids|k_inverse_plan|k_bits_emit)" \
  -s 120 -c 16 -o gpurun_out/final2/full -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final2/ncu_full.log 2>&1
