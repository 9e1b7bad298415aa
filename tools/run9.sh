set -x
mkdir -p gpurun_out/r9
for v in default nt512; do
  if [ $v = default ]; then L=paper_2506_23775_b200/libgfcuda.so; else L=paper_2506_23775_b200/variants/libgfcuda_$v.so; fi
  GF_LIB_PATH=$L timeout 600 python bench.py --summands 16384 --steps 3 --warmup 2 --no-sweep --no-cpu --no-c5 --e2e-steps 1 > gpurun_out/r9/b_$v.json 2>gpurun_out/r9/b_$v.err
  python -c "import json; d=json.load(open('gpurun_out/r9/b_$v.json')); print('$v', round(d['ms_per_step'],1), {k:(v['ms'], v.get('fp64_tflops')) for k,v in d['phases'].items()})" >> gpurun_out/r9/summary.txt
  for c in c4 c5; do
    GF_LIB_PATH=$L timeout 600 python bench_configs.py --one $c > gpurun_out/r9/${c}_$v.json 2>>gpurun_out/r9/cfg.err
    python -c "import json; d=json.load(open('gpurun_out/r9/${c}_$v.json')); print('$v $c', d['grad_hvp_s_per_summand'])" >> gpurun_out/r9/summary.txt
  done
done
cat gpurun_out/r9/summary.txt
