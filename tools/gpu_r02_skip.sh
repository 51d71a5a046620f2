# no stream wait on host jobs already finished (skip), + staging after the write-back marks only (marks), vs prev
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prefetch.py tests/test_gpu_memory.py -x -q 2>&1 | tail -2 > gpurun_out/sk_tests.txt
for i in 1 2 3 4; do
  for v in prev skip marks; do
    E=""; [ $v = prev ] && E="FC_LIB_PATH=tools/ab/lib_prev.so"; [ $v = marks ] && E="FC_XFER_AFTER_MARKS=1"
    echo "$v $(env $E timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["step_latency_ms"]; print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1), "pool", round(s["pool_avg"],3), "upd", round(s["update_avg"],3), "xfer", round(s["miss_transfer_avg"],3))')" >> gpurun_out/sk_ab.txt
  done
done
