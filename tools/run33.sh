set -x
mkdir -p gpurun_out/r33
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r33/pytest.log 2>&1; tail -n 4 gpurun_out/r33/pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-c5 > gpurun_out/r33/bench.json 2> gpurun_out/r33/bench.err
python -c "import json; a=json.load(open('gpurun_out/r33/bench.json')); print(a['value'], a['ms_per_step'], a['e2e']['value'], {k:(v['ms'],v.get('fp64_tflops')) for k,v in a['phases'].items()})"
for c in c3 c4 c5 c1; do
    timeout 600 python bench_configs.py --one $c > gpurun_out/r33/${c}.json 2>>gpurun_out/r33/cfg.err
    python -c "import json; d=json.load(open('gpurun_out/r33/${c}.json')); print('$c', d.get('grad_hvp_s_per_summand'), d.get('full_sum_grad_hvp_s'), d.get('trust_region_5_iterations_s'))"
done
