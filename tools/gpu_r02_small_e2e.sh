# small config e2e stalls: current build vs the build before the commit reorder (noclear), 3 rounds;
# e2e M lookups/s, host step p50 / max ms, device value
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in cur noclear; do
    E=""; [ $v = noclear ] && E="FC_LIB_PATH=tools/ab/lib_noclear.so"
    echo "$v $(env $E timeout 300 python bench.py --config small --steps 200 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d["e2e"]; print(round(d["value"]/1e6,1), "e2e", round(e["value"]/1e6,1), "host p50", round(e["host_step_ms"]["p50"],3), "max", round(e["host_step_ms"]["max"],2))')" >> gpurun_out/small_e2e.txt
  done
done
for v in cur noclear; do
  E=""; [ $v = noclear ] && E="FC_LIB_PATH=tools/ab/lib_noclear.so"
  echo "== $v" >> gpurun_out/small_stall.txt
  env $E FC_DEBUG_WAITS=1 timeout 300 python tools/e2e_stall.py small >> gpurun_out/small_stall.txt 2>&1
done
