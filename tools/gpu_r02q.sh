# C5 multi-GPU time split (graph wall / host-stepped wall / engine events; exchange pack vs unpack+wait) at N = 2, 4
for n in 2 4; do
  AKMC_PHASE_TIMING=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29531 \
    tools/multi_probe.py > gpurun_out/multi_probe_n$n.log 2>&1; echo n$n=$?
  grep "graph_ms\|akmc exchange" gpurun_out/multi_probe_n$n.log
done
