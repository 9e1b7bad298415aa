set -x
mkdir -p gpurun_out/r35
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r35/pytest_gpu_r02f.log 2>&1; tail -n 3 gpurun_out/r35/pytest_gpu_r02f.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r35/smoke.log 2>&1; tail -n 2 gpurun_out/r35/smoke.log
timeout 1500 python bench.py > gpurun_out/r35/bench_r02d.json 2> gpurun_out/r35/bench.err; tail -c 300 gpurun_out/r35/bench_r02d.json
timeout 1500 python bench.py --impl reference > gpurun_out/r35/bench_r02d_reference_arm.json 2>> gpurun_out/r35/bench.err
timeout 1500 python bench_configs.py c1 c3 c4 c5 c3tr c5h c2h > gpurun_out/r35/configs_r02e.jsonl 2> gpurun_out/r35/cfg.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r35/launches_bench_r02d.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-c5 --e2e-steps 1 > gpurun_out/r35/ncu_launch.log 2>&1; tail -n 2 gpurun_out/r35/ncu_launch.log
R='regex:k_fused<\(int\)3, \(bool\)1, \(int\)256, \(int\)1, \(int\)0>'
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$R" -s 3 -c 1 -o /tmp/ncu_rev1 python bench.py --steps 1 --warmup 1 --no-sweep --no-cpu --no-c5 --e2e-steps 1 --summands 8192 > gpurun_out/r35/ncu_rev1.log 2>&1; tail -n 2 gpurun_out/r35/ncu_rev1.log
ncu -i /tmp/ncu_rev1.ncu-rep --page raw --csv > gpurun_out/r35/ncu_c2_rev_first_raw.csv 2>/dev/null
timeout 900 python bench.py --gpus 2 --backend gloo --steps 2 --warmup 3 --no-sweep --no-cpu --no-c5 --summands 16384 > gpurun_out/r35/bench_gpus2_gloo.json 2>gpurun_out/r35/bench2.err; tail -c 200 gpurun_out/r35/bench_gpus2_gloo.json
du -sh gpurun_out/r35
