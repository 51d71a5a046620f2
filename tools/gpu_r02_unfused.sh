# fused backward (default) vs sums-then-apply (FC_BWD_UNFUSED=1): isolated + in the pipeline
mkdir -p gpurun_out
for i in 1 2; do
  for v in 0 1; do
    E=""; [ $v = 1 ] && E="FC_BWD_UNFUSED=1"
    echo "iso unfused=$v $(env $E timeout 300 python tools/bwd_bench.py 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_avg"]*1e3,1), "us", round(d["frac_hbm"],3))')" >> gpurun_out/unf.txt
  done
done
for i in 1 2 3; do
  for v in 0 1; do
    E=""; [ $v = 1 ] && E="FC_BWD_UNFUSED=1"
    echo "step unfused=$v $(env $E timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["step_latency_ms"]; print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1), "upd", round(s["update_avg"],3))')" >> gpurun_out/unf.txt
  done
done
