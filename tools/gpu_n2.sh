# 2-GPU: multi-rank parity tests, then the N=2 bench (watchdog on) three times
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi.log 2>&1; echo pytest_multi=$?; tail -3 gpurun_out/pytest_multi.log
for i in 1 2 3; do
  AKMC_WATCHDOG=1 timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2952$i bench.py --gpus 2 --no-cpu-baseline > gpurun_out/n2_$i.json 2> gpurun_out/n2_$i.err
  echo run=$i rc=$?
  python -c "import json;d=json.load(open('gpurun_out/n2_$i.json'));print(d['value'],d['ms_per_step'])" 2>/dev/null
  grep -i "watchdog\|akmc" gpurun_out/n2_$i.err | head -20
done
