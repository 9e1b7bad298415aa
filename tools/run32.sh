set -x
mkdir -p gpurun_out/r32
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r32/pytest.log 2>&1; tail -n 12 gpurun_out/r32/pytest.log
for v in "GF_LIGHTCONE=1" "GF_LIGHTCONE=0"; do
env $v timeout 900 python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-c5 > gpurun_out/r32/bench_$v.json 2> gpurun_out/r32/bench.err
python -c "import json; a=json.load(open('gpurun_out/r32/bench_$v.json')); print('$v', a['value'], a['ms_per_step'], a['e2e']['value'], {k:(v['ms'],v.get('fp64_tflops')) for k,v in a['phases'].items()})"
done
for c in c3 c4 c5; do
    timeout 600 python bench_configs.py --one $c > gpurun_out/r32/${c}.json 2>>gpurun_out/r32/cfg.err
    python -c "import json; d=json.load(open('gpurun_out/r32/${c}.json')); print('$c', d['grad_hvp_s_per_summand'], d.get('reinsertion_max_rel_dev'))"
done
