python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
AKMC_PHASE_TIMING=1 timeout 300 python tools/df_probe.py 4 > gpurun_out/df_probe_timing.log 2>&1; echo probe2=$?
grep -v "iter trace\]  [0-9]\|iter trace\] it" gpurun_out/df_probe_timing.log | tail -14
