set -x
mkdir -p gpurun_out/r31
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r31/pytest_gpu_r02e.log 2>&1; tail -n 3 gpurun_out/r31/pytest_gpu_r02e.log
timeout 1500 python bench.py > gpurun_out/r31/bench_r02c.json 2> gpurun_out/r31/bench.err; tail -c 300 gpurun_out/r31/bench_r02c.json
timeout 1500 python bench.py --impl reference > gpurun_out/r31/bench_r02c_reference_arm.json 2>> gpurun_out/r31/bench.err
timeout 1500 python bench_configs.py c1 c3 c4 c5 c3tr c5h c2h > gpurun_out/r31/configs_r02d.jsonl 2> gpurun_out/r31/cfg.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r31/launches_bench_r02c.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-c5 --e2e-steps 1 > gpurun_out/r31/ncu_launch.log 2>&1; tail -n 2 gpurun_out/r31/ncu_launch.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 400 --csv --log-file gpurun_out/r31/launches_c4_unit_r02c.csv python tools/c4_one.py 14 > gpurun_out/r31/ncu_l.log 2>&1
timeout 600 python bench_v1.py gradient --out gpurun_out/r31 > gpurun_out/r31/bv1.log 2>&1; tail -n 3 gpurun_out/r31/bv1.log
du -sh gpurun_out/r31
