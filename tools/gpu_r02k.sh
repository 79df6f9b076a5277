python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python tools/df_probe.py 10 > gpurun_out/df_probe.log 2>&1; echo probe=$?
timeout 300 python tools/df_probe.py 10 1.0 > gpurun_out/df_probe_lam1.log 2>&1; echo probe1=$?
AKMC_PHASE_TIMING=1 timeout 300 python tools/df_probe.py 4 > gpurun_out/df_probe_timing.log 2>&1; echo probe2=$?
AKMC_WATCHDOG=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k "fp64" -p no:cacheprovider --timeout 800 > gpurun_out/pytest_full_r02k.log 2>&1; echo full=$?
cat gpurun_out/df_probe.log gpurun_out/df_probe_lam1.log; grep "iterations/CTA\|trace\] it\|trace\]  [0-9]\|sync\|dataflow" gpurun_out/df_probe_timing.log | head -40; tail -3 gpurun_out/pytest_full_r02k.log
