# full GPU suite after the memory_report fix; row-sharded world-1 step (NCCL return) + timeline
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/full_gpu.txt
timeout 600 python bench.py --gpus 1 --shard row --no-cpu-baseline > gpurun_out/row_nccl.json 2> gpurun_out/row_nccl.err
FC_TORCH_TRACE=gpurun_out/tl_row.json timeout 300 python bench.py --gpus 1 --shard row --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tl_row.out 2>&1
python tools/timeline.py gpurun_out/tl_row.json 1 2 > gpurun_out/tl_row.txt 2>&1; gzip -f gpurun_out/tl_row.json
