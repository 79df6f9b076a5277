python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x > gpurun_out/pytest_gpu_n.log 2>&1; echo pytest=$?
timeout 300 python tools/df_probe.py 10 > gpurun_out/df_probe_n.log 2>&1; echo probe=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_n.json 2> gpurun_out/bench_n.err; echo bench=$?
tail -3 gpurun_out/pytest_gpu_n.log; cat gpurun_out/df_probe_n.log
python -c "import json; d=json.loads(open('gpurun_out/bench_n.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['evaluator_bulk']['ms'], d['e2e']['value'])"
