set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest2.log 2>&1; tail -5 gpurun_out/pytest2.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -c 600 gpurun_out/bench2.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench2_ref.json 2> gpurun_out/bench2_ref.err
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py > gpurun_out/memcheck.log 2>&1; tail -4 gpurun_out/memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 20 python tools/sanitize_case.py > gpurun_out/racecheck.log 2>&1; tail -4 gpurun_out/racecheck.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 30 -c 4 -o gpurun_out/ncu_c4 python tools/c4_one.py 14 > gpurun_out/ncu_c4.log 2>&1; tail -3 gpurun_out/ncu_c4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/c4_one.py 14 > gpurun_out/launches_c4.log 2>&1
