python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_mfpt.py tests/test_gpu_world.py -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_mfpt_r02e.log 2>&1; echo mfpt=$?
tail -15 gpurun_out/pytest_mfpt_r02e.log
