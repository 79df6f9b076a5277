python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build4.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -rs > gpurun_out/pytest_multi4.log 2>&1; echo pytest_multi=$?; tail -4 gpurun_out/pytest_multi4.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --no-cpu-baseline > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo bench4=$?
python -c "import json;d=json.load(open('gpurun_out/bench_n4.json'));print(d['value'],d['ms_per_step'],d['n_gpus'],d['config'].get('parallelism'))"
