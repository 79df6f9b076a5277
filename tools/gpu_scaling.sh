# weak scaling N = 1, 2, 4 (C5 per GPU) with the driver's launch line
for N in 1 2 4; do
  if [ $N = 1 ]; then timeout 600 python bench.py --no-cpu-baseline > gpurun_out/scale_n1.json 2> gpurun_out/scale_n1.err
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N > gpurun_out/scale_n$N.json 2> gpurun_out/scale_n$N.err; fi
  echo N=$N rc=$?
  python -c "import json;d=json.load(open('gpurun_out/scale_n$N.json'));print(d['n_gpus'],d['value'],d['ms_per_step'],d['config']['parallelism'])"
done
