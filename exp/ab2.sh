for v in lib_trim lib_plan; do
  echo "$v" >> gpurun_out/ab.log
  GF_LIB_PATH=exp/$v.so python bench.py --steps 1 --warmup 1 --no-sweep --no-cpu --e2e-steps 1 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],1), d['config'].get('engine'), {k:v['ms'] for k,v in d['phases'].items()})" >> gpurun_out/ab.log
done
