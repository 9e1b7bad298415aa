for pp in 1 0; do
  echo "pipe=$pp" >> gpurun_out/ab.log
  GF_PIPE=$pp python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --e2e-steps 1 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],1), d['config'].get('engine'), {k:v['ms'] for k,v in d['phases'].items()})" >> gpurun_out/ab.log
done
