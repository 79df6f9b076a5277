# 1 GPU: full suite after the FP32 E3/L3 arithmetic change, bulk A/B (producer warps 8 vs 16), bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu_r02i.log 2>&1; echo pytest=$?
AKMC_PHASE_TIMING=1 python tools/bulk_probe.py 5 > gpurun_out/bulk_p8.log 2>&1
AKMC_PHASE_TIMING=1 AKMC_LIB=paper_2604_24091_b200/lib/libakmc_prod16.so python tools/bulk_probe.py 5 > gpurun_out/bulk_p16.log 2>&1
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_r02i.json 2> gpurun_out/bench_r02i.err; echo bench=$?
tail -4 gpurun_out/pytest_gpu_r02i.log; grep "akmc bulk\|rep 4" gpurun_out/bulk_p8.log gpurun_out/bulk_p16.log
python -c "import json; d=json.loads(open('gpurun_out/bench_r02i.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['evaluator_bulk']['ms'], d['roofline']['evaluator_bulk']['executed_frac'])"
