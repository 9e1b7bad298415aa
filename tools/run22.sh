set -x
mkdir -p gpurun_out/r22
timeout 900 python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu --no-c5 > gpurun_out/r22/bench.json 2> gpurun_out/r22/bench.err
timeout 600 python bench_configs.py --one c5 > gpurun_out/r22/c5.json 2>>gpurun_out/r22/cfg.err
