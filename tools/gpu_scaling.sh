# weak scaling N = 1, 2, 4 (C5 per GPU, and C4 voxel batches) with the driver's launch line; multi-GPU tests
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi.log 2>&1; echo pytest_multi=$?; tail -2 gpurun_out/pytest_multi.log
for W in c5 c4; do
for N in 1 2 4; do
  if [ $N = 1 ]; then timeout 600 python bench.py --workload $W --no-cpu-baseline > gpurun_out/scale_${W}_n1.json 2> gpurun_out/scale_${W}_n1.err
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --workload $W --gpus $N > gpurun_out/scale_${W}_n$N.json 2> gpurun_out/scale_${W}_n$N.err; fi
  echo $W N=$N rc=$?
  python -c "import json;d=json.load(open('gpurun_out/scale_${W}_n$N.json'));print(d['n_gpus'],d['value'],d['ms_per_step'],d['config']['parallelism'])"
done
done
