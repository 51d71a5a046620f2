# A/B on one box: default vs FC_POOL_NO_TMA (LDG k_pool1) vs FC_WB_EXACT=0 (ship every victim), 3 rounds alternating
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in default pool_ldg wb_all; do
    case $v in
      default) E="";;
      pool_ldg) E="FC_POOL_NO_TMA=1";;
      wb_all) E="FC_WB_EXACT=0";;
    esac
    echo "$v $(env $E timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["step_latency_ms"]; print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1), "pool", round(s["pool_avg"],3), "upd", round(s["update_avg"],3), "xfer", round(s["miss_transfer_avg"],3))')" >> gpurun_out/ab_pool.txt
  done
done
