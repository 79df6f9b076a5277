# 1 GPU: dataflow correctness (watchdog aborts a hang after 20 s), then C5 timing
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
AKMC_WATCHDOG=1 timeout 600 python -m pytest tests/test_gpu_guards.py -q -k dataflow -p no:cacheprovider -x --timeout 200 > gpurun_out/pytest_df_r02j.log 2>&1; echo df=$?
tail -30 gpurun_out/pytest_df_r02j.log
AKMC_WATCHDOG=1 timeout 300 python tools/df_probe.py 10 > gpurun_out/df_probe.log 2>&1; echo probe=$?
tail -20 gpurun_out/df_probe.log
