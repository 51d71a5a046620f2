# round-2 session-3 first look: full GPU suite, default bench, column/1tb lines, reference arm, launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/r02_gpu_tests.txt
timeout 600 python bench.py > gpurun_out/r02_cfg2.json 2> gpurun_out/r02_cfg2.err
timeout 600 python bench.py --gpus 1 --shard column --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_cfg2_col.json 2> gpurun_out/r02_cfg2_col.err
timeout 900 python bench.py --config criteo_1tb --gpus 1 --shard column --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_1tb_col.json 2> gpurun_out/r02_1tb_col.err
timeout 600 python bench.py --impl reference > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
