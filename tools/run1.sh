set -x
python -c "import __graft_entry__ as g; g.build()"
for v in 0 1; do for c in c3 c4 c5; do GF_SPARSE_DMMA=$v timeout 600 python bench_configs.py --one $c > gpurun_out/cfg_$c_$v.json 2>gpurun_out/cfg_err_$c_$v.log; echo "SPARSE_DMMA=$v $c" >> gpurun_out/cfg_summary.txt; cat gpurun_out/cfg_$c_$v.json >> gpurun_out/cfg_summary.txt; done; done
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest1.log 2>&1; tail -3 gpurun_out/pytest1.log
