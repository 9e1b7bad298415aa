mkdir -p gpurun_out/r43
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r43/pytest_gpu_r02g.log 2>&1; tail -n 3 gpurun_out/r43/pytest_gpu_r02g.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -n 1
