# A/B of library builds on a 4096-summand slice of the c2 bench
for v in "$@"; do
  for rep in 1 2; do
    echo "$v rep$rep" >> gpurun_out/ab.log
    GF_LIB_PATH=exp/$v.so python bench.py --summands 4096 --steps 3 --warmup 1 --no-sweep --no-cpu --e2e-steps 1 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],1), {k:v['ms'] for k,v in d['phases'].items()})" >> gpurun_out/ab.log
  done
done
