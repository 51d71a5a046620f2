mkdir -p gpurun_out/san
FC_XFER_TMA=0 FC_NO_TMA=1 timeout 900 compute-sanitizer --tool initcheck --print-limit 10 python -m pytest tests/test_gpu_prefetch.py -q -x -k "module_prefetch and adagrad" > gpurun_out/san/initcheck_notma.log 2>&1; echo rc=$? >> gpurun_out/san/initcheck_notma.log
