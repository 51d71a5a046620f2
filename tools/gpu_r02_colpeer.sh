# fused column exchange: GPU tests, then column-wise cfg2 at world 1 with and without --peer (alternating)
mkdir -p gpurun_out/colpeer; rm -f gpurun_out/colpeer/*
timeout 900 python -m pytest tests/test_gpu_column.py -q -x 2>&1 | tail -2
for i in 1 2; do
  timeout 600 python bench.py --gpus 1 --shard column --no-cpu-baseline > gpurun_out/colpeer/nccl_$i.json 2>/dev/null
  timeout 600 python bench.py --gpus 1 --shard column --peer --no-cpu-baseline > gpurun_out/colpeer/peer_$i.json 2>gpurun_out/colpeer/peer_$i.err
done
for f in gpurun_out/colpeer/*.json; do python -c "
import json; d=json.load(open('$f')); e=d.get('e2e') or {}
print('$f'.split('/')[-1], round(d['value']/1e6,1), round(d['ms_per_step'],3), round(e['value']/1e6,1), d['implementation']['exchange'][:40])" 2>&1 | tail -1; done
tail -3 gpurun_out/colpeer/peer_1.err
