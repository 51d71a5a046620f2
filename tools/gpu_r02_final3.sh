# round-2 closing evidence on the current build: GPU suite + smoke, bench lines (cfg2 x2, small,
# avazu, stress, column/row/table at world 1, criteo_1tb column), reference arm, ncu launch list
mkdir -p gpurun_out/final3
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/final3/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final3/smoke.txt 2>&1
for i in 1 2; do timeout 600 python bench.py > gpurun_out/final3/cfg2_$i.json 2> gpurun_out/final3/cfg2_$i.err; done
for c in small avazu stress; do timeout 900 python bench.py --config $c > gpurun_out/final3/$c.json 2> gpurun_out/final3/$c.err; done
for sh in column row table; do
  timeout 600 python bench.py --gpus 1 --shard $sh --no-cpu-baseline > gpurun_out/final3/cfg2_$sh.json 2> gpurun_out/final3/cfg2_$sh.err
done
timeout 900 python bench.py --config criteo_1tb --gpus 1 --shard column --no-cpu-baseline > gpurun_out/final3/1tb_col.json 2> gpurun_out/final3/1tb_col.err
timeout 600 python bench.py --impl reference > gpurun_out/final3/ref.json 2> gpurun_out/final3/ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final3/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
cat gpurun_out/final3/gpu_tests.txt gpurun_out/final3/smoke.txt
for f in gpurun_out/final3/*.json; do python -c "
import json; d=json.load(open('$f')); e=d.get('e2e') or {}; r=d.get('roofline') or {}
print('$f'.split('/')[-1], round(d['value']/1e6,1), round(d.get('ms_per_step',0),3), round((e.get('value') or 0)/1e6,1), r.get('frac'), (d.get('clocks') or {}).get('reasons'))" 2>&1 | tail -1; done
