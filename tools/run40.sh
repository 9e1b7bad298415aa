mkdir -p gpurun_out/r40
for v in "GF_PLAN_MINPASS=1" "GF_X=1" "GF_PLAN_MINPASS=1" "GF_X=1"; do
env $v timeout 900 python bench.py --steps 4 --warmup 3 --no-sweep --no-cpu --no-c5 --e2e-steps 2 > gpurun_out/r40/bench_$v.json 2> gpurun_out/r40/bench.err
python -c "import json; a=json.load(open('gpurun_out/r40/bench_$v.json')); print('$v', a['value'], a['ms_per_step'], a['e2e']['value'], a['roofline']['frac'], a['engine']['rev_passes'], sum(v['ms'] for v in a['phases'].values())/a['steps'])"
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r40/pytest.log 2>&1; tail -n 3 gpurun_out/r40/pytest.log
for c in c3 c4 c5; do
    timeout 600 python bench_configs.py --one $c > gpurun_out/r40/${c}.json 2>>gpurun_out/r40/cfg.err
    python -c "import json; d=json.load(open('gpurun_out/r40/${c}.json')); print('$c', d.get('grad_hvp_s_per_summand'), d['engine'])"
done
