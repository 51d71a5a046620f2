# paced miss staging: prefetch parity tests, then an in-pipeline rate sweep at cfg2 (FC_XFER_GBPS, 0 = unpaced)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_prefetch.py tests/test_gpu_column.py -x -q 2>&1 | tail -2 > gpurun_out/pace_tests.txt
for i in 1 2; do
  for r in 0 30 33 36 39; do
    echo "gbps=$r $(FC_XFER_GBPS=$r timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["step_latency_ms"]; print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1), "pool", round(s["pool_avg"],3), "upd", round(s["update_avg"],3), "xfer", round(s["miss_transfer_avg"],3))')" >> gpurun_out/pace_sweep.txt
  done
done
FC_TORCH_TRACE=gpurun_out/tl_pace.json timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tl_pace.out 2>&1
python tools/timeline.py gpurun_out/tl_pace.json 1 2 > gpurun_out/tl_pace.txt 2>&1; gzip -f gpurun_out/tl_pace.json
