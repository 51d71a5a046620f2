mkdir -p gpurun_out
python -m pytest tests/test_gpu_prefetch.py -x -q -k "clean_victims or two_ahead or depth2" 2>&1 | tail -3 > gpurun_out/r02_wb_tests.txt
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02_wb_a$i.json 2> gpurun_out/r02_wb_a$i.err; done
FC_WB_EXACT=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02_wb_x.json 2> gpurun_out/r02_wb_x.err
