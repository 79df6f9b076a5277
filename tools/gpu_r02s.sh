# overlapped exchange (side stream: unpack + boundary activation; engine runs interior domains first): 2 ranks
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -x -k "two_rank" > gpurun_out/pytest_multi_ov2.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_multi_ov2.log
for n in 2; do
  AKMC_PHASE_TIMING=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29531 \
    tools/multi_probe.py > gpurun_out/multi_probe_ov_n$n.log 2>&1; echo n$n=$?
  grep "graph_ms\|akmc exchange" gpurun_out/multi_probe_ov_n$n.log
  AKMC_OVERLAP=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29531 \
    tools/multi_probe.py > gpurun_out/multi_probe_noov_n$n.log 2>&1; echo n$n=$?
  grep "graph_ms" gpurun_out/multi_probe_noov_n$n.log
done
