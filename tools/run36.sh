set -x
mkdir -p gpurun_out/r36
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r36/pytest.log 2>&1; tail -n 3 gpurun_out/r36/pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-c5 > gpurun_out/r36/bench.json 2> gpurun_out/r36/bench.err
python -c "import json; a=json.load(open('gpurun_out/r36/bench.json')); print(a['value'], a['ms_per_step'], a['e2e']['value'], a['roofline']['frac'], a['engine']['oracle_setup_s'], {k:(v['ms'],v.get('fp64_tflops')) for k,v in a['phases'].items()})"
for c in c4 c5; do
    timeout 600 python bench_configs.py --one $c > gpurun_out/r36/${c}.json 2>>gpurun_out/r36/cfg.err
    python -c "import json; d=json.load(open('gpurun_out/r36/${c}.json')); print('$c', d.get('grad_hvp_s_per_summand'), d.get('oracle_s_per_summand'))"
done
