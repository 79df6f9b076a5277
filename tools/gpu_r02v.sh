# fused send+receive exchange kernel (one launch per phase): 2-rank tests + C5 timing, then N = 2 bench line
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider -x -k "two_rank or overlapped" > gpurun_out/pytest_multi_fx.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_multi_fx.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/multi_probe.py 2>&1 | grep graph_ms
timeout 600 python bench.py --workload c5 --no-cpu-baseline > gpurun_out/scale_c5_n1.json 2> gpurun_out/scale_c5_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --workload c5 --gpus 2 > gpurun_out/scale_c5_n2.json 2> gpurun_out/scale_c5_n2.err
for n in 1 2; do python -c "import json;d=json.load(open('gpurun_out/scale_c5_n$n.json'));print(d['n_gpus'],d['value'],d['ms_per_step'])"; done
