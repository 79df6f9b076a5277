# round 2b: new tests first (bulk evaluator, guards), then the full GPU suite, smoke, bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_guards.py -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_guards_r02b.log 2>&1; echo guards=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu_r02b.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 400 python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo bench=$?
tail -12 gpurun_out/pytest_guards_r02b.log; tail -12 gpurun_out/pytest_gpu_r02b.log; tail -2 gpurun_out/smoke.log; tail -c 1500 gpurun_out/bench_r02b.json; tail -5 gpurun_out/bench_r02b.err
