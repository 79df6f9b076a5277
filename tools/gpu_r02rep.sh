# flakiness check at HEAD: the multi-rank tests twice more and the whole suite once, 4-GPU box
for rep in 1 2; do
  timeout 1500 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/rep_multi$rep.log 2>&1; echo multi$rep=$?; tail -1 gpurun_out/rep_multi$rep.log
done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/rep_all.log 2>&1; echo all=$?; tail -1 gpurun_out/rep_all.log
