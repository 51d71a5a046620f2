mkdir -p gpurun_out
rm -f gpurun_out/fused.txt
for i in 1 2 3; do for v in X=1 FC_BWD_UNFUSED=1; do
  env $v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_v.json 2> /dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_v.json')); print('$v', round(d['value']/1e6,1), round(d['ms_per_step'],3), round(d['e2e']['value']/1e6,1))" >> gpurun_out/fused.txt
done; done
