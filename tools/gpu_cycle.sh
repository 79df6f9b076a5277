python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
AKMC_PHASE_TIMING=1 timeout 300 python tools/iter_probe.py --cells 1024 --sweeps 4 --no-rates > gpurun_out/iter.log 2>&1
tail -22 gpurun_out/iter.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline']['evaluator_bulk']['ms'])"
