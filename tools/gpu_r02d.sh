python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_world.py tests/test_gpu_guards.py -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_world_r02d.log 2>&1; echo world=$?
python tools/bulk_probe.py 5 > gpurun_out/bulk_probe.log 2>&1; echo probe=$?
AKMC_EVAL_ENGINE=1 python tools/bulk_probe.py 3 > gpurun_out/bulk_probe_engine.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bulk_eval -s 2 -c 1 -o gpurun_out/prof_bulk -f python tools/bulk_probe.py 3 > gpurun_out/ncu_bulk.log 2>&1; echo ncu=$?
tail -15 gpurun_out/pytest_world_r02d.log; cat gpurun_out/bulk_probe.log gpurun_out/bulk_probe_engine.log; tail -3 gpurun_out/ncu_bulk.log
