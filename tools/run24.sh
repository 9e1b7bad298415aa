set -x
mkdir -p gpurun_out/r24
for v in "GF_X=0" "GF_DIRS_PER_SWEEP=1"; do
  env $v timeout 900 python bench_configs.py --one c5h > gpurun_out/r24/c5h_$v.json 2>>gpurun_out/r24/cfg.err
  python -c "import json; d=json.load(open('gpurun_out/r24/c5h_$v.json')); print('$v c5h', {k:d.get(k) for k in ('gradient_s_per_summand','hvp20_s_per_summand','directions_per_sweep','gradient_plus_20_hvp_s_per_summand','multi_vs_single_hvp_max_rel_dev')})" >> gpurun_out/r24/summary.txt
done
for v in "GF_X=0" "GF_DIRS_PER_SWEEP=1"; do
  env $v timeout 900 python bench_configs.py --one c3tr > gpurun_out/r24/c3tr_$v.json 2>>gpurun_out/r24/cfg.err
  python -c "import json; d=json.load(open('gpurun_out/r24/c3tr_$v.json')); print('$v c3tr', {k:v for k,v in d.items() if 's_per' in k or 'tr_' in k})" >> gpurun_out/r24/summary.txt
done
cat gpurun_out/r24/summary.txt; tail -n 3 gpurun_out/r24/cfg.err
