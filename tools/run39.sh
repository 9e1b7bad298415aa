mkdir -p gpurun_out/r39
for v in "GF_PLAN_MINPASS=1" "GF_X=1"; do
env $v timeout 900 python bench.py --steps 4 --warmup 3 --no-sweep --no-cpu --no-c5 --e2e-steps 1 > gpurun_out/r39/bench_$v.json 2> gpurun_out/r39/bench.err
python -c "import json; a=json.load(open('gpurun_out/r39/bench_$v.json')); print('$v', a['value'], a['ms_per_step'], a['engine']['live_fraction'], a['engine']['rev_passes'], {k:v['ms'] for k,v in a['phases'].items()})"
done
timeout 900 python -m pytest tests -m gpu -x -q -k "config or engine or planner or checked" > gpurun_out/r39/pytest.log 2>&1; tail -n 3 gpurun_out/r39/pytest.log
