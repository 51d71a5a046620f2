# 4-way A/B on one box: prev (round-2 HEAD before these), chain (staging waits only for the write-back
# marks + no stream wait on finished host jobs), fused (11-launch index phase only), both
mkdir -p gpurun_out
run() {
  echo "$1 $(env $2 timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["step_latency_ms"]; print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1), "pool", round(s["pool_avg"],3), "upd", round(s["update_avg"],3), "xfer", round(s["miss_transfer_avg"],3))')" >> gpurun_out/ab4.txt
}
for i in 1 2 3; do
  run prev "FC_LIB_PATH=tools/ab/lib_prev.so"
  run chain "FC_LIB_PATH=tools/ab/lib_chain.so"
  run fused "FC_XFER_WAIT_COMMIT=1 FC_ALWAYS_WAIT_JOB=1"
  run both ""
done
