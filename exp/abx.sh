# A/B: exp/base.so (HEAD) vs the working-tree libgfcuda.so on the c2 bench step
run() { echo "$1 | $2" >> gpurun_out/ab.log; env $1 python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu --e2e-steps 1 $2 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],1), {k:v['ms'] for k,v in d['phases'].items()}, 'frac', d['roofline']['frac'], 'e2e', round(d['e2e']['value'],4))" >> gpurun_out/ab.log; }
for cfg in "$@"; do run "$cfg" ""; done
