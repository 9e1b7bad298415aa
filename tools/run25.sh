set -x
mkdir -p gpurun_out/r25
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r25/pytest_gpu_r02d.log 2>&1; tail -n 3 gpurun_out/r25/pytest_gpu_r02d.log
timeout 1500 python bench.py > gpurun_out/r25/bench_r02b.json 2> gpurun_out/r25/bench.err; tail -c 600 gpurun_out/r25/bench_r02b.json
timeout 1500 python bench.py --impl reference > gpurun_out/r25/bench_r02b_reference_arm.json 2>> gpurun_out/r25/bench.err
timeout 1500 python bench_configs.py c1 c3 c4 c5 c3tr c5h > gpurun_out/r25/configs_r02c.jsonl 2> gpurun_out/r25/cfg.err
NT=256
R="regex:k_fused<\(int\)3, \(bool\)0, \(int\)$NT, \(int\)1, \(int\)4>"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$R" -s 2 -c 1 -o /tmp/ncu_unit python tools/c4_one.py 14 > gpurun_out/r25/ncu_unit.log 2>&1; tail -n 2 gpurun_out/r25/ncu_unit.log
ncu -i /tmp/ncu_unit.ncu-rep --page raw --csv > gpurun_out/r25/ncu_c4_unit_rev_raw.csv 2>/dev/null
ncu -i /tmp/ncu_unit.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r25/ncu_c4_unit_rev_source.csv 2>/dev/null
gzip -f gpurun_out/r25/ncu_c4_unit_rev_source.csv
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 400 --csv --log-file gpurun_out/r25/launches_c4_unit_r02.csv python tools/c4_one.py 14 > gpurun_out/r25/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "$R" -s 2 -c 1 -o /tmp/ncu_c5 python tools/c4_one.py 16 > gpurun_out/r25/ncu_c5.log 2>&1; tail -n 2 gpurun_out/r25/ncu_c5.log
ncu -i /tmp/ncu_c5.ncu-rep --page raw --csv > gpurun_out/r25/ncu_c5_unit_rev_raw.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r25/launches_bench_r02b.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-c5 --e2e-steps 1 > gpurun_out/r25/ncu_launch.log 2>&1; tail -n 2 gpurun_out/r25/ncu_launch.log
du -sh gpurun_out/r25
