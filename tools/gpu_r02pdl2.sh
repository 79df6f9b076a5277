# PDL also for the activate / segments kernels (engine triggers its dependents at exit): parity + A/B
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "not multi" > gpurun_out/pytest_pdl2.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_pdl2.log
for rep in 1 2; do
for v in "" _nopdl2; do
  if [ -n "$v" ]; then export AKMC_LIB=paper_2604_24091_b200/lib/libakmc$v.so; else unset AKMC_LIB; fi
  for w in c5 c3; do
    timeout 600 python bench.py --workload $w --no-cpu-baseline --steps 20 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pdl2$v', $rep, '$w', d['value'], d['ms_per_step'])"
  done
done
done
