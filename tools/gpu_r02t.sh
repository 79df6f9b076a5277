# overlap timing (boundary-list publication vs engine start), 2 ranks
AKMC_PHASE_TIMING=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
    tools/multi_probe.py > gpurun_out/multi_probe_ovt_n2.log 2>&1; echo n2=$?
grep "graph_ms\|akmc overlap\|akmc exchange\|akmc engine\] CTA" gpurun_out/multi_probe_ovt_n2.log
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -x -k "two_rank" > gpurun_out/pytest_multi_ov2.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_multi_ov2.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/multi_probe.py 2>&1 | grep graph_ms
AKMC_OVERLAP=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/multi_probe.py 2>&1 | grep graph_ms
