# weak scaling N = 1, 2, 4 of C5 at lambda = 1 (4x the events per phase of the default 1/4)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for N in 1 2 4; do
  if [ $N = 1 ]; then timeout 600 python bench.py --lam 1.0 --no-cpu-baseline > gpurun_out/scale_l1_n1.json 2> gpurun_out/scale_l1_n1.err
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --lam 1.0 --gpus $N > gpurun_out/scale_l1_n$N.json 2> gpurun_out/scale_l1_n$N.err; fi
  echo N=$N rc=$?
  python -c "import json;d=json.load(open('gpurun_out/scale_l1_n$N.json'));print(d['n_gpus'],d['value'],d['ms_per_step'],d['events_per_s'],d['sim_seconds_per_wall_second'])"
done
