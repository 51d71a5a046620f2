# isolated fused backward at cfg2 for backward-stream shapes chunk_unroll_minblocks (tools/build_bwd_variants.sh)
mkdir -p gpurun_out
for i in 1 2; do
  for v in 64_4_4 32_4_4 128_4_4 64_4_3 32_4_3 64_8_3 64_8_4 32_8_4 128_8_3 64_4_6; do
    echo "$v $(FC_LIB_PATH=tools/ab/bwd_$v.so timeout 300 python tools/bwd_bench.py 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_avg"]*1e3,1), "us", round(d["frac_hbm"],3), "rel_err", d["max_rel_err_vs_f64"])')" >> gpurun_out/bwd_sweep.txt
  done
done
