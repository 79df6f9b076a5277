# bulk evaluator (10 producer warps, b1' in shared memory, branch-free E3): tests, timing, ncu --set full of one call
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x -k "bulk or eval_windows or rates" > gpurun_out/pytest_bulk4.log 2>&1; echo pytest=$?
tail -1 gpurun_out/pytest_bulk4.log
timeout 300 python tools/bulk_probe.py 8 > gpurun_out/bulk4t.log 2>&1; echo probe=$?
grep rep gpurun_out/bulk4t.log | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk_eval -s 2 -c 1 -o gpurun_out/prof_bulk4 \
  python tools/bulk_probe.py 3 > gpurun_out/ncu_bulk4.log 2>&1; echo ncu=$?
