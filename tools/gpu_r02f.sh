# 4-GPU box: multi-rank tests (2 and 4 ranks), new single-GPU tests, scheduling A/B, weak scaling 1/2/4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
nvidia-smi -L > gpurun_out/smi_L.txt
timeout 1800 python -m pytest tests/test_gpu_multi.py -v -p no:cacheprovider --timeout 900 > gpurun_out/pytest_multi_r02f.log 2>&1; echo multi=$?
timeout 600 python -m pytest tests/test_gpu_guards.py -q -k voxel -p no:cacheprovider > gpurun_out/pytest_order_r02f.log 2>&1; echo order=$?
python tools/sched_probe.py 40000 > gpurun_out/sched_r02f.log 2>&1; AKMC_VOXEL_FIFO=1 python tools/sched_probe.py 40000 >> gpurun_out/sched_r02f.log 2>&1; echo sched=$?
for N in 1 2 4; do
  if [ $N = 1 ]; then timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/scale_c5_n1.json 2> gpurun_out/scale_c5_n1.err;
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2950$N bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/scale_c5_n$N.json 2> gpurun_out/scale_c5_n$N.err; fi
  echo scale$N=$?
done
for N in 2 4; do AKMC_EXCHANGE=shift timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/scale_c5_shift_n$N.json 2> gpurun_out/scale_c5_shift_n$N.err; echo shift$N=$?; done
grep -E "PASS|FAIL|SKIP|passed|failed" gpurun_out/pytest_multi_r02f.log | tail -25; tail -3 gpurun_out/pytest_order_r02f.log; cat gpurun_out/sched_r02f.log
for f in gpurun_out/scale_c5_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'])" 2>/dev/null || echo "$f bad"; done
