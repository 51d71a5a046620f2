mkdir -p gpurun_out
python -m pytest tests/test_gpu_column.py -x -q 2>&1 | tail -15 > gpurun_out/r02_col_tests.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_cfg2.json 2> gpurun_out/r02_cfg2.err
timeout 600 python bench.py --gpus 1 --shard column --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_cfg2_col.json 2> gpurun_out/r02_cfg2_col.err
timeout 600 python bench.py --gpus 1 --shard row --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_cfg2_row.json 2> gpurun_out/r02_cfg2_row.err
timeout 900 python bench.py --config criteo_1tb --gpus 1 --shard column --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_1tb_col.json 2> gpurun_out/r02_1tb_col.err
timeout 600 python bench.py --impl reference --steps 4 --warmup 2 > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err
