# eviction commit without waiting for the staging (next stage freed by the previous commit, 4 write-back
# stages): GPU suite, A/B vs the previous build (4 rounds), timeline
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pc2_tests.txt
for i in 1 2 3 4 5; do
  for v in prev new; do
    E=""; [ $v = prev ] && E="FC_LIB_PATH=tools/ab/lib_prev.so"
    echo "$v $(env $E timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["step_latency_ms"]; print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1), "pool", round(s["pool_avg"],3), "upd", round(s["update_avg"],3), "xfer", round(s["miss_transfer_avg"],3))')" >> gpurun_out/pc2_ab.txt
  done
done
FC_TORCH_TRACE=gpurun_out/tl_pc2.json timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tl_pc2.out 2>&1
python tools/timeline.py gpurun_out/tl_pc2.json 1 2 > gpurun_out/tl_pc2.txt 2>&1; gzip -f gpurun_out/tl_pc2.json
