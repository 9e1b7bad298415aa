set -x
mkdir -p gpurun_out/r21
export GF_FUSED_PERSIST=0
for c in c4 c5; do
    timeout 600 python bench_configs.py --one $c > gpurun_out/r21/${c}.json 2>>gpurun_out/r21/cfg.err
    python -c "import json; d=json.load(open('gpurun_out/r21/${c}.json')); print('$c', d['grad_hvp_s_per_summand'], d.get('reinsertion_max_rel_dev'))" >> gpurun_out/r21/summary.txt
done
cat gpurun_out/r21/summary.txt
timeout 900 python bench.py --steps 4 --warmup 3 --no-sweep --no-cpu --no-c5 > gpurun_out/r21/bench.json 2> gpurun_out/r21/bench.err
