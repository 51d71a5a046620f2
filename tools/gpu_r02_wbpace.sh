# write-back D2H pacing experiment (copier ships the dirty rows in 4 MB pieces at a capped rate)
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in default exact p40 p30 p20; do
    case $v in default) E="";; exact) E="FC_WB_EXACT=1";; p40) E="FC_WB_EXACT=1 FC_WB_PACE_GBPS=40";; p30) E="FC_WB_EXACT=1 FC_WB_PACE_GBPS=30";; p20) E="FC_WB_EXACT=1 FC_WB_PACE_GBPS=20";; esac
    echo "$v $(env $E timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["step_latency_ms"]; print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1), "pool", round(s["pool_avg"],3), "upd", round(s["update_avg"],3), "xfer", round(s["miss_transfer_avg"],3))')" >> gpurun_out/wbp_ab.txt
  done
done
