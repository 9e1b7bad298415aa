set -x
mkdir -p gpurun_out/r18
NT=256
R="regex:k_fused<\(int\)3, \(bool\)0, \(int\)$NT, \(int\)1, \(int\)4>"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$R" -s 2 -c 1 -o /tmp/ncu_unit$NT python tools/c4_one.py 14 > gpurun_out/r18/ncu_unit$NT.log 2>&1; tail -n 2 gpurun_out/r18/ncu_unit$NT.log
ncu -i /tmp/ncu_unit$NT.ncu-rep --page raw --csv > gpurun_out/r18/ncu_unit${NT}_rev_raw.csv 2>/dev/null
ncu -i /tmp/ncu_unit$NT.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r18/ncu_unit${NT}_rev_source.csv 2>/dev/null
gzip -f gpurun_out/r18/ncu_unit${NT}_rev_source.csv
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 400 --csv --log-file gpurun_out/r18/launches_c4_unit.csv python tools/c4_one.py 14 > gpurun_out/r18/ncu_l.log 2>&1
