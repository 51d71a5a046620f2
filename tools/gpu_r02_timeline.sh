# pipelined cfg2 step timelines (CUPTI via torch.profiler) with and without the miss staging
mkdir -p gpurun_out
FC_TORCH_TRACE=gpurun_out/tl_default.json timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tl_default.out 2>&1
FC_DEBUG_SKIP_STAGING=1 FC_TORCH_TRACE=gpurun_out/tl_nostage.json timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tl_nostage.out 2>&1
for f in default nostage; do python tools/timeline.py gpurun_out/tl_$f.json 1 2 > gpurun_out/tl_$f.txt 2>&1; gzip -f gpurun_out/tl_$f.json; done
timeout 600 python -m pytest tests/test_gpu_column.py -x -q 2>&1 | tail -3 > gpurun_out/col_tests.txt
timeout 600 python bench.py --gpus 1 --shard column --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/col_pf.json 2> gpurun_out/col_pf.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/cfg2_ldg.json 2> gpurun_out/cfg2_ldg.err
