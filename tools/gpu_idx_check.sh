mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
FC_XFER_AFTER_UPDATE=1 timeout 200 python tools/pipeline_timeline.py --steps 10 --index-stream side > gpurun_out/timeline_defer.txt 2>&1
timeout 200 python tools/pipeline_timeline.py --steps 10 --index-stream side > gpurun_out/timeline_side.txt 2>&1
