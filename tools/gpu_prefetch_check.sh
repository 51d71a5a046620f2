mkdir -p gpurun_out
export CUDA_DEVICE_MAX_CONNECTIONS=32
for m in main side; do for x in 64 96 148; do FC_XFER_BLOCKS=$x timeout 200 python tools/pipeline_timeline.py --steps 12 --index-stream $m > gpurun_out/timeline_${m}_$x.txt 2>&1; done; done
