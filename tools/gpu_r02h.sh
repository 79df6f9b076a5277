# 2-GPU box: bulk v1 role timing (1 GPU), then the 2-rank C5 bench (p2p) three times, no watchdog, bounded
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
AKMC_PHASE_TIMING=1 python tools/bulk_probe.py 5 > gpurun_out/bulk_probe1.log 2>&1; echo probe=$?
for k in 1 2 3; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$k bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/scale_c5_n2_$k.json 2> gpurun_out/scale_c5_n2_$k.err; echo scale2_$k=$?
done
grep "akmc bulk\|rep " gpurun_out/bulk_probe1.log
for k in 1 2 3; do python -c "import json; d=json.loads(open('gpurun_out/scale_c5_n2_$k.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])" 2>/dev/null || (echo "run $k failed"; grep -v "^  " gpurun_out/scale_c5_n2_$k.err | tail -5); done
