for cfg in "11 16 64" "11 32 64" "11 32 37" "11 16 74" "12 8 64" "12 16 64" "10 32 64" "10 64 64"; do
  set -- $cfg
  echo "m=$1 ctas=$2 batch=$3" >> gpurun_out/tune.log
  GF_FUSED_M=$1 GF_FUSED_CTAS=$2 python bench.py --summands 4096 --batch $3 --steps 2 --warmup 1 --no-sweep --no-cpu --e2e-steps 1 2>>gpurun_out/tune.err | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['ms_per_step'],1), {k:(v['ms'],v['launches']) for k,v in d['phases'].items()})" >> gpurun_out/tune.log
done
