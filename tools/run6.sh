set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out/r6
timeout 1800 python -m pytest tests -q -m gpu -x -k "hessian or integration or pair or kernels or checked or non_finite or array or hole" > gpurun_out/r6/pytest6.log 2>&1; tail -5 gpurun_out/r6/pytest6.log
for c in c2hp bw16d; do timeout 900 python bench_configs.py --one $c >> gpurun_out/r6/cfg6.txt 2>>gpurun_out/r6/cfg6.err; done
timeout 600 python bench_v1.py kernels --qubits 20,24,26 --repeats 5 --out gpurun_out/r6 > gpurun_out/r6/bv6.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 2 --no-sweep --no-cpu --no-c5 > gpurun_out/r6/bench6.json 2> gpurun_out/r6/bench6.err
R='regex:k_fused<\(int\)3, \(bool\)0, \(int\)256, \(int\)1, \(int\)0>'
C='regex:k_fused<\(int\)3, \(bool\)0, \(int\)256, \(int\)1, \(int\)2>'
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$R" -s 4 -c 1 -o /tmp/ncu_rev python bench.py --steps 1 --warmup 1 --no-sweep --no-cpu --no-c5 --e2e-steps 1 --summands 4096 > gpurun_out/r6/ncu_rev.log 2>&1; tail -n 2 gpurun_out/r6/ncu_rev.log
ncu -i /tmp/ncu_rev.ncu-rep --page raw --csv > gpurun_out/r6/ncu_rev_raw.csv 2>/dev/null
ncu -i /tmp/ncu_rev.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r6/ncu_rev_source.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "$C" -s 2 -c 1 -o /tmp/ncu_c5 python tools/c4_one.py 16 > gpurun_out/r6/ncu_c5.log 2>&1; tail -n 2 gpurun_out/r6/ncu_c5.log
ncu -i /tmp/ncu_c5.ncu-rep --page raw --csv > gpurun_out/r6/ncu_c5rev_raw.csv 2>/dev/null
du -sh gpurun_out
