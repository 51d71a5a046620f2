# after the commit reorder: the next staging waits only for the write-back marks (new) vs the whole commit
# (FC_XFER_AFTER_COMMIT=1, same build) vs the committed build (prev); parity suites first
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_prefetch.py tests/test_gpu_memory.py tests/test_gpu_column.py tests/test_gpu_simulator.py -x -q 2>&1 | tail -2 > gpurun_out/mk_tests.txt
for i in 1 2 3 4; do
  for v in prev commit new; do
    E=""; [ $v = prev ] && E="FC_LIB_PATH=tools/ab/lib_prev.so"; [ $v = commit ] && E="FC_XFER_AFTER_COMMIT=1"
    echo "$v $(env $E timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["step_latency_ms"]; print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1), "pool", round(s["pool_avg"],3), "upd", round(s["update_avg"],3), "xfer", round(s["miss_transfer_avg"],3), "mhz", d["clocks"]["sm_mhz"])')" >> gpurun_out/mk_ab.txt
  done
done
FC_TORCH_TRACE=gpurun_out/tl_mk.json timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tl_mk.out 2>&1
python tools/timeline.py gpurun_out/tl_mk.json 1 2 > gpurun_out/tl_mk.txt 2>&1; gzip -f gpurun_out/tl_mk.json
