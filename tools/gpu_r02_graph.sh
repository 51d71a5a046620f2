# the pipeline's index phase as one CUDA-graph launch (FC_INDEX_GRAPH=1) vs kernel by kernel:
# parity suites with the graph on, A/B on one box, a timeline with the graph on
mkdir -p gpurun_out
FC_INDEX_GRAPH=1 timeout 1200 python -m pytest tests/test_gpu_prefetch.py tests/test_gpu_memory.py tests/test_gpu_column.py tests/test_gpu_simulator.py tests/test_gpu_embedding.py -x -q 2>&1 | tail -2 > gpurun_out/gr_tests.txt
for i in 1 2 3 4; do
  for v in 0 1; do
    echo "graph=$v $(FC_INDEX_GRAPH=$v timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["step_latency_ms"]; print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1), "pool", round(s["pool_avg"],3), "upd", round(s["update_avg"],3), "xfer", round(s["miss_transfer_avg"],3))')" >> gpurun_out/gr_ab.txt
  done
done
for c in small avazu; do
  for v in 0 1; do
    echo "$c graph=$v $(FC_INDEX_GRAPH=$v timeout 600 python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e6,1), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,1))')" >> gpurun_out/gr_ab.txt
  done
done
FC_INDEX_GRAPH=1 FC_TORCH_TRACE=gpurun_out/tl_gr.json timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tl_gr.out 2>&1
python tools/timeline.py gpurun_out/tl_gr.json 1 2 > gpurun_out/tl_gr.txt 2>&1; gzip -f gpurun_out/tl_gr.json
