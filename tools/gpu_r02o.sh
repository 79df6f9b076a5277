# bulk evaluator: default (10 producers, TMEM prefetch, branch-free E3) vs _p8 = no prefetch, _p12 = no prefetch + 8 producers
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x -k "bulk or eval_windows or rates" > gpurun_out/pytest_bulk3.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_bulk3.log
for v in "" _p8 _p12; do
  if [ -n "$v" ]; then export AKMC_LIB=paper_2604_24091_b200/lib/libakmc$v.so; fi
  AKMC_PHASE_TIMING=1 timeout 300 python tools/bulk_probe.py 5 > gpurun_out/bulk3$v.log 2>&1; echo probe$v=$?
  timeout 300 python tools/bulk_probe.py 8 > gpurun_out/bulk3t$v.log 2>&1
done
unset AKMC_LIB
AKMC_LIB=paper_2604_24091_b200/lib/libakmc_p12.so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x -k "bulk" > gpurun_out/pytest_bulk3_p12.log 2>&1; echo pytest12=$?
for v in "" _p8 _p12; do echo "== $v"; grep -h "akmc bulk" gpurun_out/bulk3$v.log; grep -h rep gpurun_out/bulk3t$v.log | tail -4; done
