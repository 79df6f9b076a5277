# GPU MFPT solver timing vs scipy BiCGSTAB (same preconditioner) on synthetic AKMC-shaped spaces
timeout 900 python -m pytest tests/test_gpu_mfpt.py -q -p no:cacheprovider > gpurun_out/pytest_mfpt.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_mfpt.log
timeout 900 python tools/mfpt_probe.py 16384 131072 1048576 > gpurun_out/mfpt_probe.log 2>&1; echo probe=$?
cat gpurun_out/mfpt_probe.log
