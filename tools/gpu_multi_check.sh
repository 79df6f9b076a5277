python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build2.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -rs > gpurun_out/pytest_multi.log 2>&1; echo pytest_multi=$?; tail -6 gpurun_out/pytest_multi.log
