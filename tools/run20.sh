set -x
mkdir -p gpurun_out/r20
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r20/pytest.log 2>&1; tail -n 5 gpurun_out/r20/pytest.log
for c in c3 c4 c5; do
    timeout 600 python bench_configs.py --one $c > gpurun_out/r20/${c}.json 2>>gpurun_out/r20/cfg.err
    python -c "import json; d=json.load(open('gpurun_out/r20/${c}.json')); print('$c', d['grad_hvp_s_per_summand'], d.get('reinsertion_max_rel_dev'))" >> gpurun_out/r20/summary.txt
done
cat gpurun_out/r20/summary.txt
timeout 900 python bench.py --steps 4 --warmup 3 --no-sweep --no-cpu --no-c5 > gpurun_out/r20/bench.json 2> gpurun_out/r20/bench.err; tail -c 1500 gpurun_out/r20/bench.json
