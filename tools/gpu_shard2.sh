mkdir -p gpurun_out
for pf in "" "--no-peer"; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --sharded --steps 10 --warmup 3 --no-cpu-baseline $pf > gpurun_out/bench_sh$pf.json 2> gpurun_out/bench_sh$pf.err
done
