set -x
mkdir -p gpurun_out/r23
timeout 900 python -m pytest tests -m gpu -x -q -k "sector or config or checked or fold or c1q" > gpurun_out/r23/pytest.log 2>&1; tail -n 3 gpurun_out/r23/pytest.log
for v in "GF_X=0" "GF_FWD_M=12"; do
  for c in c4 c5; do
    env $v timeout 600 python bench_configs.py --one $c > gpurun_out/r23/${c}_$v.json 2>>gpurun_out/r23/cfg.err
    python -c "import json; d=json.load(open('gpurun_out/r23/${c}_$v.json')); print('$v $c', d['grad_hvp_s_per_summand'], d.get('reinsertion_max_rel_dev'), d['engine'])" >> gpurun_out/r23/summary.txt
  done
done
for v in 16 8; do
GF_FUSED_CTAS=$v timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu --no-c5 --e2e-steps 1 > gpurun_out/r23/bench_ctas$v.json 2> gpurun_out/r23/bench.err
python -c "import json; a=json.load(open('gpurun_out/r23/bench_ctas$v.json')); print('ctas $v', a['value'], a['ms_per_step'], {k:(v['ms'],v.get('fp64_tflops')) for k,v in a['phases'].items()})" >> gpurun_out/r23/summary.txt
done
cat gpurun_out/r23/summary.txt
