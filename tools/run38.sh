set -x
mkdir -p gpurun_out/r38
timeout 1500 python bench.py > gpurun_out/r38/bench_r02e.json 2> gpurun_out/r38/bench.err; tail -c 200 gpurun_out/r38/bench_r02e.json
timeout 1500 python bench.py --impl reference > gpurun_out/r38/bench_r02e_reference_arm.json 2>> gpurun_out/r38/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1200 --csv --log-file gpurun_out/r38/launches_bench_r02e.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-c5 --e2e-steps 1 > gpurun_out/r38/ncu_launch.log 2>&1; tail -n 2 gpurun_out/r38/ncu_launch.log
R='regex:k_fused<\(int\)3, \(bool\)1, \(int\)256, \(int\)1, \(int\)0>'
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$R" -s 3 -c 1 -o /tmp/ncu_rev1 python bench.py --steps 1 --warmup 1 --no-sweep --no-cpu --no-c5 --e2e-steps 1 --summands 8192 > gpurun_out/r38/ncu_rev1.log 2>&1; tail -n 2 gpurun_out/r38/ncu_rev1.log
ncu -i /tmp/ncu_rev1.ncu-rep --page raw --csv > gpurun_out/r38/ncu_c2_rev_first_raw.csv 2>/dev/null
timeout 600 python bench_v1.py kernels --qubits 20,24 --repeats 5 --out gpurun_out/r38 > gpurun_out/r38/bv.log 2>&1; tail -n 2 gpurun_out/r38/bv.log
