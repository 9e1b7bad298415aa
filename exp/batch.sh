for b in 16 32 48 64; do
  echo "trim batch=$b" >> gpurun_out/ab.log
  GF_LIB_PATH=exp/lib_trim.so python bench.py --batch $b --steps 1 --warmup 1 --no-sweep --no-cpu --e2e-steps 1 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],1), {k:v['ms'] for k,v in d['phases'].items()})" >> gpurun_out/ab.log
done
