set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1800 python -m pytest tests -q -m gpu -x -k "sector or fold or multi_tile or c3 or c4 or c5 or folded or hessian or integration or c1" > gpurun_out/pytest3.log 2>&1; tail -15 gpurun_out/pytest3.log
rm -f gpurun_out/cfg3.txt
for c in c3 c4 c5; do timeout 600 python bench_configs.py --one $c >> gpurun_out/cfg3.txt 2>>gpurun_out/cfg3.err; done
for c in c3 c4; do GF_C1Q_DMMA=0 timeout 600 python bench_configs.py --one $c >> gpurun_out/cfg3_fma.txt 2>>gpurun_out/cfg3.err; done
timeout 600 python bench_configs.py --one c2h >> gpurun_out/cfg3.txt 2>>gpurun_out/cfg3.err
tail -3 gpurun_out/cfg3.err
