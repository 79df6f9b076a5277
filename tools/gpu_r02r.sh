# p2p exchange with warp-aggregated reservations, one fence per block, 16 blocks: multi-rank tests + timing split
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_multi_r02r.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_multi_r02r.log
bash tools/gpu_r02q.sh
