set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest4.log 2>&1; tail -5 gpurun_out/pytest4.log
rm -f gpurun_out/cfg4.txt
for c in c2hp bw16d c3tr c5h; do timeout 900 python bench_configs.py --one $c >> gpurun_out/cfg4.txt 2>>gpurun_out/cfg4.err; done
timeout 600 python bench_v1.py kernels --qubits 12,20,24,26,28 --repeats 5 --out gpurun_out > gpurun_out/bv1.log 2>&1
timeout 600 python bench_v1.py gradient --qubits 12,16 --layers 5 --inits 2 --out gpurun_out >> gpurun_out/bv1.log 2>&1
timeout 600 python bench_v1.py hessian --qubits 10,12 --layers 5 --inits 2 --bench-dedup --out gpurun_out >> gpurun_out/bv1.log 2>&1
tail -3 gpurun_out/cfg4.err
