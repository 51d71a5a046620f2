# backward without its histogram kernel (digit histograms made by the pipeline's k_unique_info):
# full GPU suite, A/B vs the previous build (3 rounds), a timeline
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/hi_tests.txt
for i in 1 2 3; do
  for v in new prev; do
    E=""; [ $v = prev ] && E="FC_LIB_PATH=tools/ab/lib_prev.so"
    echo "$v $(env $E timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["step_latency_ms"]; print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1), "pool", round(s["pool_avg"],3), "upd", round(s["update_avg"],3), "xfer", round(s["miss_transfer_avg"],3))')" >> gpurun_out/hi_ab.txt
  done
done
FC_TORCH_TRACE=gpurun_out/tl_hi.json timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tl_hi.out 2>&1
python tools/timeline.py gpurun_out/tl_hi.json 1 2 > gpurun_out/tl_hi.txt 2>&1; gzip -f gpurun_out/tl_hi.json
