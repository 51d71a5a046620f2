# every config's bench line on the current build + a small-config timeline
mkdir -p gpurun_out
for c in small avazu stress; do
  timeout 900 python bench.py --config $c > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
done
timeout 900 python bench.py --config criteo_1tb --gpus 1 --shard column --no-cpu-baseline > gpurun_out/cfg_1tb_col.json 2> gpurun_out/cfg_1tb_col.err
timeout 600 python bench.py --gpus 1 --shard row --no-cpu-baseline > gpurun_out/cfg_row1.json 2> gpurun_out/cfg_row1.err
FC_TORCH_TRACE=gpurun_out/tl_small.json timeout 300 python bench.py --config small --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tl_small.out 2>&1
python tools/timeline.py gpurun_out/tl_small.json 3 2 > gpurun_out/tl_small.txt 2>&1; gzip -f gpurun_out/tl_small.json
