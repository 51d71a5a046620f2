#!/bin/bash
# round 2: compute-sanitizer memcheck / racecheck over the fused index phase, the histogram
# ring, the commit reorder and the bounded (tiny, growing) stages
mkdir -p gpurun_out/san2
timeout 1500 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_memory.py tests/test_gpu_prefetch.py -q -x -k "tiny_stages or depth2 or (random_parity and 3000) or sync_prepare_into or paced" > gpurun_out/san2/memcheck.log 2>&1; echo rc=$? >> gpurun_out/san2/memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_prefetch.py tests/test_gpu_embedding.py -q -x -k "(random_parity and 3000 and 1) or sequence_of_batch_sizes" > gpurun_out/san2/racecheck.log 2>&1; echo rc=$? >> gpurun_out/san2/racecheck.log
timeout 1500 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_gpu_prefetch.py -q -x -k "random_parity and 3000 and 2" > gpurun_out/san2/synccheck.log 2>&1; echo rc=$? >> gpurun_out/san2/synccheck.log
for f in gpurun_out/san2/*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $f | tail -4; done > gpurun_out/san2/summary.txt
