# 2-GPU box: bulk v2 correctness + timing (1 GPU), then the 2-rank C5 bench (p2p) under a watchdog
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_guards.py -q -k "bulk or crowded or large_activ or overflow or resume" -p no:cacheprovider --timeout 300 > gpurun_out/pytest_bulk2_r02g.log 2>&1; echo bulktests=$?
AKMC_PHASE_TIMING=1 python tools/bulk_probe.py 5 > gpurun_out/bulk_probe2.log 2>&1; echo probe=$?
AKMC_WATCHDOG=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29502 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/scale_c5_n2b.json 2> gpurun_out/scale_c5_n2b.err; echo scale2=$?
tail -5 gpurun_out/pytest_bulk2_r02g.log; cat gpurun_out/bulk_probe2.log | grep -v "^\[akmc iter\|engine" | tail -8
tail -c 400 gpurun_out/scale_c5_n2b.json; grep -v "^  " gpurun_out/scale_c5_n2b.err | tail -20
