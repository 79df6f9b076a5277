# multi-rank sweep as one CUDA graph (device-side exchange epoch): all multi tests, then C5 scaling N = 1, 2, 4
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/pytest_multi_gr.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_multi_gr.log
for N in 1 2 4; do
  if [ $N = 1 ]; then timeout 600 python bench.py --workload c5 --no-cpu-baseline > gpurun_out/scale_c5_n1g.json 2> gpurun_out/scale_c5_n1g.err
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --workload c5 --gpus $N > gpurun_out/scale_c5_n${N}g.json 2> gpurun_out/scale_c5_n${N}g.err; fi
  python -c "import json;d=json.load(open('gpurun_out/scale_c5_n${N}g.json'));print(d['n_gpus'],d['value'],d['ms_per_step'],d['gpu_launches'])"
done
