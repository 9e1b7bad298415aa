set -x
mkdir -p gpurun_out/r12
export GF_UNIT_NT=256
python tools/c4_one.py 14 > gpurun_out/r12/plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 400 --csv --log-file gpurun_out/r12/launches_c4_unit.csv python tools/c4_one.py 14 > gpurun_out/r12/ncu_l.log 2>&1
R='regex:k_fused<\(int\)3, \(bool\)0, \(int\)256, \(int\)1, \(int\)4>'
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$R" -s 2 -c 1 -o /tmp/ncu_unit python tools/c4_one.py 14 > gpurun_out/r12/ncu_unit.log 2>&1; tail -n 2 gpurun_out/r12/ncu_unit.log
ncu -i /tmp/ncu_unit.ncu-rep --page raw --csv > gpurun_out/r12/ncu_unit_rev_raw.csv 2>/dev/null
ncu -i /tmp/ncu_unit.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r12/ncu_unit_rev_source.csv 2>/dev/null
gzip -f gpurun_out/r12/ncu_unit_rev_source.csv
for v in "GF_SECTOR_FMA=0" "GF_SECTOR_FMA=1"; do
  env $v GF_EXP_NOIO=1 timeout 600 python bench_configs.py --one c4 > gpurun_out/r12/c4_noio_$v.json 2>>gpurun_out/r12/cfg.err
  python -c "import json; d=json.load(open('gpurun_out/r12/c4_noio_$v.json')); print('NOIO $v c4', d['grad_hvp_s_per_summand'])" >> gpurun_out/r12/summary.txt
  env $v GF_EXP_NOSLOTS=1 timeout 600 python bench_configs.py --one c4 > gpurun_out/r12/c4_noslots_$v.json 2>>gpurun_out/r12/cfg.err
  python -c "import json; d=json.load(open('gpurun_out/r12/c4_noslots_$v.json')); print('NOSLOTS $v c4', d['grad_hvp_s_per_summand'])" >> gpurun_out/r12/summary.txt
done
cat gpurun_out/r12/summary.txt
