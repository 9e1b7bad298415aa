set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
mkdir -p gpurun_out/r8
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r8/pytest8.log 2>&1; tail -5 gpurun_out/r8/pytest8.log
for c in c2hp bw16d; do timeout 900 python bench_configs.py --one $c >> gpurun_out/r8/cfg8.txt 2>>gpurun_out/r8/cfg8.err; done
timeout 600 python bench_v1.py kernels --qubits 20,24,26 --repeats 5 --out gpurun_out/r8 > gpurun_out/r8/bv8.log 2>&1
