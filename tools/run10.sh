set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out/r10
timeout 1800 python -m pytest tests -q -m gpu -x -k "sector or fold or multi_tile or c3 or c4 or c5 or folded or multi_direction or checked or c1 or c2" > gpurun_out/r10/pytest.log 2>&1; tail -5 gpurun_out/r10/pytest.log
for v in 1 0; do for c in c3 c4 c5; do
  GF_PAIR_BLOCKS=$v timeout 600 python bench_configs.py --one $c > gpurun_out/r10/${c}_$v.json 2>>gpurun_out/r10/cfg.err
  python -c "import json; d=json.load(open('gpurun_out/r10/${c}_$v.json')); print('pair=$v $c', d['grad_hvp_s_per_summand'], d['hvp_s_per_summand'], d['reinsertion_max_rel_dev'])" >> gpurun_out/r10/summary.txt
done; done
cat gpurun_out/r10/summary.txt
