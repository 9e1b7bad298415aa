mkdir -p gpurun_out/r37
for i in 1 2; do
timeout 900 python bench.py --no-sweep --no-cpu --no-c5 > gpurun_out/r37/bench_def$i.json 2> gpurun_out/r37/bench.err
python -c "import json; a=json.load(open('gpurun_out/r37/bench_def$i.json')); print('default', a['steps'], a['warmup'], a['value'], a['ms_per_step'], a['e2e']['value'], a['roofline']['frac'], sum(v['ms'] for v in a['phases'].values())/a['steps'])"
timeout 900 python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-c5 > gpurun_out/r37/bench_5_$i.json 2> gpurun_out/r37/bench.err
python -c "import json; a=json.load(open('gpurun_out/r37/bench_5_$i.json')); print('5/3', a['steps'], a['warmup'], a['value'], a['ms_per_step'], a['e2e']['value'], a['roofline']['frac'], sum(v['ms'] for v in a['phases'].values())/a['steps'])"
done
