# write-back stage count: 4 (committed) vs 6 vs 8, cfg2 + avazu + stress; then the GPU suite on the 6-stage build
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in d4 s6 s8; do
    case $v in d4) L=tools/ab/lib_default4.so;; s6) L=tools/ab/lib_s6.so;; s8) L=tools/ab/lib_s8.so;; esac
    echo "$v $(FC_LIB_PATH=$L timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["step_latency_ms"]; print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1), "upd", round(s["update_avg"],3), "xfer", round(s["miss_transfer_avg"],3))')" >> gpurun_out/stages_ab.txt
  done
done
for c in avazu stress; do
  for v in d4 s6 s8; do
    case $v in d4) L=tools/ab/lib_default4.so;; s6) L=tools/ab/lib_s6.so;; s8) L=tools/ab/lib_s8.so;; esac
    echo "$c $v $(FC_LIB_PATH=$L timeout 600 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1))')" >> gpurun_out/stages_ab.txt
  done
done
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/stages_tests.txt
