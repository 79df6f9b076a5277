# HEAD multi-GPU: all multi-rank tests (incl. AKMC_OVERLAP=1), then C5 weak scaling N = 1, 2, 4 (driver launch line)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/pytest_multi_r02u.log 2>&1; echo pytest_multi=$?; tail -2 gpurun_out/pytest_multi_r02u.log
for N in 1 2 4; do
  if [ $N = 1 ]; then timeout 600 python bench.py --workload c5 --no-cpu-baseline > gpurun_out/scale_c5_n1.json 2> gpurun_out/scale_c5_n1.err
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --workload c5 --gpus $N > gpurun_out/scale_c5_n$N.json 2> gpurun_out/scale_c5_n$N.err; fi
  echo N=$N rc=$?
  python -c "import json;d=json.load(open('gpurun_out/scale_c5_n$N.json'));print(d['n_gpus'],d['value'],d['ms_per_step'],d['e2e']['value'])"
done
