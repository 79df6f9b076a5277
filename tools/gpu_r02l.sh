python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
AKMC_WATCHDOG=1 timeout 600 python -m pytest tests/test_gpu_guards.py -q -k dataflow -p no:cacheprovider -x --timeout 200 > gpurun_out/pytest_df_r02l.log 2>&1; echo df=$?
tail -5 gpurun_out/pytest_df_r02l.log
timeout 300 python tools/df_probe.py 10 > gpurun_out/df_probe.log 2>&1; echo probe=$?
AKMC_PHASE_TIMING=1 timeout 300 python tools/df_probe.py 4 > gpurun_out/df_probe_timing.log 2>&1; echo probe2=$?
cat gpurun_out/df_probe.log; grep "CTA-launches\|trace\]  [0-9]" gpurun_out/df_probe_timing.log | head -30
