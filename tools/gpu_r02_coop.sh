# cooperative one-launch backward: parity tests, isolated A/B, in-pipeline A/B (FC_BWD_MULTI=1 = old 7-launch path)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_embedding.py tests/test_gpu_prefetch.py tests/test_gpu_router.py tests/test_gpu_peer.py tests/test_gpu_column.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -5 > gpurun_out/coop_tests.txt
for v in coop multi; do
  E=""; [ $v = multi ] && E="FC_BWD_MULTI=1"
  echo "$v $(env $E timeout 300 python tools/bwd_bench.py 2>&1 | tail -1)" >> gpurun_out/coop_iso.txt
done
for i in 1 2; do
  for v in coop multi; do
    E=""; [ $v = multi ] && E="FC_BWD_MULTI=1"
    echo "$v $(env $E timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["step_latency_ms"]; print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1), "pool", round(s["pool_avg"],3), "upd", round(s["update_avg"],3), "xfer", round(s["miss_transfer_avg"],3))')" >> gpurun_out/coop_ab.txt
  done
done
FC_TORCH_TRACE=gpurun_out/tl_coop.json timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tl_coop.out 2>&1
python tools/timeline.py gpurun_out/tl_coop.json 1 2 > gpurun_out/tl_coop.txt 2>&1; gzip -f gpurun_out/tl_coop.json
