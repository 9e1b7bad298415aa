run() { echo "$1" >> gpurun_out/ab.log; env $1 python bench.py --steps 1 --warmup 1 --no-sweep --no-cpu --e2e-steps 1 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],1), d['config'].get('engine'), {k:v['ms'] for k,v in d['phases'].items()})" >> gpurun_out/ab.log; }
run "GF_PIPE=1 GF_SEG_TILES=8"
run "GF_PIPE=1 GF_SEG_TILES=64"
run "GF_PIPE=1 GF_FUSED_M=11 GF_SEG_TILES=8"
run "GF_PIPE=0"
