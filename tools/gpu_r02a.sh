# round 2: full GPU suite (no -x), smoke, default bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu_r02a.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 400 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo bench=$?
tail -15 gpurun_out/pytest_gpu_r02a.log; tail -2 gpurun_out/smoke.log; tail -c 600 gpurun_out/bench_r02a.json
