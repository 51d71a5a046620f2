mkdir -p gpurun_out
rm -f gpurun_out/dbg_full.txt
for i in 1 2; do timeout 600 python -m pytest tests -m gpu -q -p no:randomly 2>&1 | grep -E "passed|failed|FAILED" >> gpurun_out/dbg_full.txt; done
