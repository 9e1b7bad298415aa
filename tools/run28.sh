mkdir -p gpurun_out/r28
for i in 1 2; do for c in c4 c3; do
    timeout 600 python bench_configs.py --one $c > gpurun_out/r28/${c}_$i.json 2>>gpurun_out/r28/cfg.err
    python -c "import json; d=json.load(open('gpurun_out/r28/${c}_$i.json')); print('$c', d['grad_hvp_s_per_summand'], d['sample_summands'])"
done; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 400 --csv --log-file gpurun_out/r28/launches_c4.csv python tools/c4_one.py 14 > gpurun_out/r28/ncu_l.log 2>&1
