# 5 more alternating rounds: backward without the histogram kernel (new) vs with (prev)
mkdir -p gpurun_out
for i in 1 2 3 4 5; do
  for v in prev new; do
    E=""; [ $v = prev ] && E="FC_LIB_PATH=tools/ab/lib_prev.so"
    echo "$v $(env $E timeout 300 python bench.py --steps 80 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["step_latency_ms"]; print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1), "pool", round(s["pool_avg"],3), "upd", round(s["update_avg"],3), "xfer", round(s["miss_transfer_avg"],3))')" >> gpurun_out/hi_ab2.txt
  done
done
