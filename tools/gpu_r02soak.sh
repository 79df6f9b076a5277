# multi-GPU soak at HEAD: long runs (many exchange epochs) of the decomposition vs 1 rank, FP32 MLP and FP64 pair
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29641 tools/multi_check.py --grid 2 2 1 --cells 32 32 32 --nvac 400 --sweeps 400 --model mlp --precision fp32 --out gpurun_out/soak_fp32.json > gpurun_out/soak_fp32.log 2>&1; echo fp32=$?
python -c "import json; d=json.load(open('gpurun_out/soak_fp32.json')); print({k: d[k] for k in d if k in ('ok','events','sweeps')})"
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29642 tools/multi_check.py --grid 1 2 2 --cells 24 24 24 --domain 6 6 6 --nvac 300 --sweeps 300 --out gpurun_out/soak_fp64.json > gpurun_out/soak_fp64.log 2>&1; echo fp64=$?
python -c "import json; d=json.load(open('gpurun_out/soak_fp64.json')); print({k: d[k] for k in d if k in ('ok','events','sweeps')})"
