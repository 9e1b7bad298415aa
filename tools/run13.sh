set -x
mkdir -p gpurun_out/r13
timeout 900 python -m pytest tests -m gpu -x -q -k "sector or config or checked or fold or c1q" > gpurun_out/r13/pytest.log 2>&1; tail -5 gpurun_out/r13/pytest.log
GF_UNIT_NT=128 timeout 600 python -m pytest tests -m gpu -x -q -k "sector or config or checked or fold or c1q" > gpurun_out/r13/pytest128.log 2>&1; tail -5 gpurun_out/r13/pytest128.log
for v in "GF_UNIT_NT=128" "GF_UNIT_NT=256"; do
  for c in c3 c4 c5; do
    env $v timeout 600 python bench_configs.py --one $c > gpurun_out/r13/${c}_$v.json 2>>gpurun_out/r13/cfg.err
    python -c "import json; d=json.load(open('gpurun_out/r13/${c}_$v.json')); print('$v $c', d['grad_hvp_s_per_summand'], d.get('reinsertion_max_rel_dev'))" >> gpurun_out/r13/summary.txt
  done
done
cat gpurun_out/r13/summary.txt
tail -5 gpurun_out/r13/cfg.err
