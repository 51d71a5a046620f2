# A/B on one box: the round-1 library (build/ab/lib_r01.so) against the current one, alternating
mkdir -p gpurun_out
for i in 1 2; do
  FC_LIB_PATH=$PWD/build/ab/lib_r01.so timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_old_$i.json 2> gpurun_out/ab_old_$i.err
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_new_$i.json 2> gpurun_out/ab_new_$i.err
done
python -m pytest tests/test_gpu_prefetch.py -x -q -k "clean_victims" 2>&1 | grep -B5 Error | head -30 > gpurun_out/r02_wb_tests.txt
