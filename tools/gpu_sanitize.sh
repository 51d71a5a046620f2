#!/bin/bash
# compute-sanitizer passes over the prefetch pipeline (depth 1 and 2). initcheck runs with the
# TMA staging off: the bulk-copy engine's shared->global stores are not tracked by initcheck
# (false "uninitialized" reports on the staged rows). The remaining initcheck reports are all
# the pipeline commit's write-back D2H, which copies an upper bound (every victim) of the
# stage because the dirty count is only known on the device; the clean victims' stage rows
# are never written and the host scatter reads only the device-counted rows.
mkdir -p gpurun_out/san
FC_XFER_TMA=0 FC_NO_TMA=1 timeout 900 compute-sanitizer --tool initcheck --print-limit 10 python -m pytest tests/test_gpu_prefetch.py -q -x -k "module_prefetch and adagrad" > gpurun_out/san/initcheck_notma.log 2>&1; echo rc=$? >> gpurun_out/san/initcheck_notma.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_prefetch.py -q -x -k "depth2 or (random_parity and 3000)" > gpurun_out/san/memcheck_depth2.log 2>&1; echo rc=$? >> gpurun_out/san/memcheck_depth2.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_prefetch.py -q -x -k "depth2_limits" > gpurun_out/san/racecheck_depth2.log 2>&1; echo rc=$? >> gpurun_out/san/racecheck_depth2.log
for f in gpurun_out/san/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|passed|failed|rc=" $f | tail -4; done
