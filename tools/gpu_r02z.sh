# C5 weak scaling at HEAD (fused tagged exchange), driver launch line, N = 1, 2, 4 -- twice for the spread
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in a b; do
for N in 1 2 4; do
  if [ $N = 1 ]; then timeout 600 python bench.py --workload c5 --no-cpu-baseline > gpurun_out/scale_c5_n1$rep.json 2> gpurun_out/scale_c5_n1$rep.err
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --workload c5 --gpus $N > gpurun_out/scale_c5_n$N$rep.json 2> gpurun_out/scale_c5_n$N$rep.err; fi
  python -c "import json;d=json.load(open('gpurun_out/scale_c5_n$N$rep.json'));print('$rep',d['n_gpus'],d['value'],d['ms_per_step'])"
done
done
