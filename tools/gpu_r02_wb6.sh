# 6 write-back stages + paced exact write-back vs the default build (4 stages, whole-stage D2H)
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in d4 s6 s6p40 s6p30; do
    case $v in d4) E="FC_LIB_PATH=tools/ab/lib_default4.so";; s6) E="";; s6p40) E="FC_WB_EXACT=1 FC_WB_PACE_GBPS=40";; s6p30) E="FC_WB_EXACT=1 FC_WB_PACE_GBPS=30";; esac
    echo "$v $(env $E timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["step_latency_ms"]; print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1), "pool", round(s["pool_avg"],3), "upd", round(s["update_avg"],3), "xfer", round(s["miss_transfer_avg"],3), "wait", round(s["async_writeback_wait_avg"],3))')" >> gpurun_out/wb6_ab.txt
  done
done
