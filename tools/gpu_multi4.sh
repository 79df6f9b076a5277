python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -k "four_rank" > gpurun_out/pytest_multi4.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_multi4.log
