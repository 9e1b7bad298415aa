set -x
mkdir -p gpurun_out/r11
timeout 900 python -m pytest tests -m gpu -x -q -k "sector or config or checked or fold or c1q or engine" > gpurun_out/r11/pytest.log 2>&1; tail -15 gpurun_out/r11/pytest.log
for v in "GF_SECTOR_FMA=0" "GF_SECTOR_FMA=1 GF_UNIT_NT=128" "GF_SECTOR_FMA=1 GF_UNIT_NT=256"; do
  for c in c3 c4 c5; do
    tag=$(echo $v | tr ' =' '__')
    env $v timeout 600 python bench_configs.py --one $c > gpurun_out/r11/${c}_$tag.json 2>>gpurun_out/r11/cfg.err
    python -c "import json; d=json.load(open('gpurun_out/r11/${c}_$tag.json')); print('$v $c', d['grad_hvp_s_per_summand'], {k:v for k,v in d.items() if 'err' in k or 'identity' in k})" >> gpurun_out/r11/summary.txt
  done
done
cat gpurun_out/r11/summary.txt
tail -5 gpurun_out/r11/cfg.err
