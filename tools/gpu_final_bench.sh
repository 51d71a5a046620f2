mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/fb_cfg2.json 2> gpurun_out/fb_cfg2.err
timeout 600 python bench.py --no-prefetch --no-cpu-baseline > gpurun_out/fb_cfg2_sync.json 2> gpurun_out/fb_cfg2_sync.err
timeout 600 python bench.py --config small > gpurun_out/fb_small.json 2> gpurun_out/fb_small.err
timeout 600 python bench.py --config avazu > gpurun_out/fb_avazu.json 2> gpurun_out/fb_avazu.err
FC_XFER_AFTER_UPDATE=1 timeout 600 python bench.py --config avazu --no-cpu-baseline > gpurun_out/fb_avazu_d1.json 2> gpurun_out/fb_avazu_d1.err
timeout 900 python bench.py --config stress > gpurun_out/fb_stress.json 2> gpurun_out/fb_stress.err
timeout 600 python bench.py --step sim --no-cpu-baseline > gpurun_out/fb_cfg2_sim.json 2> gpurun_out/fb_cfg2_sim.err
timeout 600 python bench.py --impl reference > gpurun_out/fb_ref.json 2> gpurun_out/fb_ref.err
