# isolated backward A/B: the in-tree library vs tools/ab/lib_r02base.so (a build of an earlier
# commit), plus the backward parity tests and a launch list of the backward kernels
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_embedding.py tests/test_gpu_prefetch.py tests/test_gpu_router.py tests/test_gpu_peer.py -x -q 2>&1 | tail -3 > gpurun_out/bwd_tests.txt
for i in 1 2; do
  for lib in paper_2208_05321_b200/libfreqcache_b200.so tools/ab/lib_r02base.so; do
    echo "lib=$lib $(FC_LIB_PATH=$lib timeout 300 python tools/bwd_bench.py 2>>gpurun_out/bwd_err.txt)" >> gpurun_out/bwd_ab.txt
  done
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_bwd|k_os|k_run" -c 40 --csv --log-file gpurun_out/bwd_launches.csv python tools/bwd_bench.py --steps 5 > /dev/null 2>&1
