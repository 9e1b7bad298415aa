run() { echo "$1" >> gpurun_out/ab.log; env $1 python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --e2e-steps 1 $2 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],1), d['config'].get('engine'), d['config']['batch'], {k:v['ms'] for k,v in d['phases'].items()}, 'e2e', d['e2e']['value'])" >> gpurun_out/ab.log; }
run "GF_PIPE=0" "--batch 128"
run "GF_PIPE=0" "--batch 256"
run "GF_PIPE=0" "--batch 64"
