set -x
mkdir -p gpurun_out/r44
R='regex:k_fused<\(int\)4, \(bool\)0, \(int\)256, \(int\)1, \(int\)0>'
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "$R" -s 8 -c 1 -f -o /tmp/ncu_asc python bench.py --steps 1 --warmup 1 --no-sweep --no-cpu --no-c5 --e2e-steps 1 --summands 8192 > gpurun_out/r44/ncu_asc.log 2>&1; tail -n 2 gpurun_out/r44/ncu_asc.log
ncu -i /tmp/ncu_asc.ncu-rep --page raw --csv > gpurun_out/r44/ncu_c2_asc_raw.csv 2>/dev/null
