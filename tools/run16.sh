set -x
mkdir -p gpurun_out/r16
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 400 --csv --log-file gpurun_out/r16/launches_c4_unit.csv python tools/c4_one.py 14 > gpurun_out/r16/ncu_l.log 2>&1
GF_SECTOR_FMA=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 400 --csv --log-file gpurun_out/r16/launches_c4_dmma.csv python tools/c4_one.py 14 > gpurun_out/r16/ncu_l0.log 2>&1
