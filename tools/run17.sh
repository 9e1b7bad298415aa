set -x
mkdir -p gpurun_out/r17
timeout 900 python -m pytest tests -m gpu -x -q -k "sector or config or checked or fold or c1q" > gpurun_out/r17/pytest.log 2>&1; tail -n 5 gpurun_out/r17/pytest.log
for v in "GF_UNIT_NT=128" "GF_UNIT_NT=256"; do
  for c in c3 c4 c5; do
    env $v timeout 600 python bench_configs.py --one $c > gpurun_out/r17/${c}_$v.json 2>>gpurun_out/r17/cfg.err
    python -c "import json; d=json.load(open('gpurun_out/r17/${c}_$v.json')); print('$v $c', d['grad_hvp_s_per_summand'], d.get('reinsertion_max_rel_dev'))" >> gpurun_out/r17/summary.txt
  done
done
cat gpurun_out/r17/summary.txt
tail -n 5 gpurun_out/r17/cfg.err
NT=256
R="regex:k_fused<\(int\)3, \(bool\)0, \(int\)$NT, \(int\)1, \(int\)4>"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$R" -s 2 -c 1 -o /tmp/ncu_unit$NT python tools/c4_one.py 14 > gpurun_out/r17/ncu_unit$NT.log 2>&1; tail -n 2 gpurun_out/r17/ncu_unit$NT.log
ncu -i /tmp/ncu_unit$NT.ncu-rep --page raw --csv > gpurun_out/r17/ncu_unit${NT}_rev_raw.csv 2>/dev/null
ncu -i /tmp/ncu_unit$NT.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r17/ncu_unit${NT}_rev_source.csv 2>/dev/null
gzip -f gpurun_out/r17/ncu_unit${NT}_rev_source.csv
