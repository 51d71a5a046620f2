mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --sharded --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sharded.json 2> gpurun_out/bench_sharded.err; echo "rc=$?" >> gpurun_out/bench_sharded.err
dmesg 2>/dev/null | tail -5 >> gpurun_out/bench_sharded.err
