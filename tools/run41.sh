set -x
mkdir -p gpurun_out/r41
timeout 1500 python bench.py > gpurun_out/r41/bench_r02f.json 2> gpurun_out/r41/bench.err; tail -c 200 gpurun_out/r41/bench_r02f.json
timeout 1500 python bench.py --impl reference > gpurun_out/r41/bench_r02f_reference_arm.json 2>> gpurun_out/r41/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r41/launches_bench_r02f.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-c5 --e2e-steps 1 > gpurun_out/r41/ncu_launch.log 2>&1; tail -n 2 gpurun_out/r41/ncu_launch.log
timeout 1500 python bench_configs.py c1 c3 c4 c5 c3tr c5h c2h > gpurun_out/r41/configs_r02f.jsonl 2> gpurun_out/r41/cfg.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r41/smoke.log 2>&1; tail -n 1 gpurun_out/r41/smoke.log
