# round-2 baseline: current state of the cfg2 bench on a fresh box
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_smi.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02_base_cfg2.json 2> gpurun_out/r02_base_cfg2.err
