python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "anisotropic" > gpurun_out/pytest_aniso.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_aniso.log
