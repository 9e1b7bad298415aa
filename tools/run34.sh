mkdir -p gpurun_out/r34
for b in 512 1024 2048 4096; do
timeout 900 python bench.py --steps 4 --warmup 3 --no-sweep --no-cpu --no-c5 --e2e-steps 2 --batch $b > gpurun_out/r34/bench_b$b.json 2> gpurun_out/r34/bench.err
python -c "import json; a=json.load(open('gpurun_out/r34/bench_b$b.json')); print('batch $b', a['value'], a['ms_per_step'], a['e2e']['value'], {k:v['ms'] for k,v in a['phases'].items()})"
done
