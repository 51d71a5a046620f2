# staging launched after the pooled forward (FC_XFER_AFTER_POOL=1) vs beside it: parity + A/B
mkdir -p gpurun_out
FC_XFER_AFTER_POOL=1 timeout 900 python -m pytest tests/test_gpu_prefetch.py tests/test_gpu_memory.py -x -q 2>&1 | tail -2 > gpurun_out/ap_tests.txt
for i in 1 2 3; do
  for v in 0 1; do
    echo "after_pool=$v $(FC_XFER_AFTER_POOL=$v timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["step_latency_ms"]; print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1), "pool", round(s["pool_avg"],3), "upd", round(s["update_avg"],3), "xfer", round(s["miss_transfer_avg"],3))')" >> gpurun_out/ap_ab.txt
  done
done
for c in avazu stress; do
  for v in 0 1; do
    echo "$c after_pool=$v $(FC_XFER_AFTER_POOL=$v timeout 600 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1))')" >> gpurun_out/ap_ab.txt
  done
done
