# engine layer 1: 4 rows per warp call with one W1' row each in flight (default) vs 2 rows x 2 (A/B), + parity tests
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "not multi" > gpurun_out/pytest_l1.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_l1.log
for rep in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/b_l141_$rep.json 2>/dev/null
  AKMC_LIB=paper_2604_24091_b200/lib/libakmc_l122.so timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/b_l122_$rep.json 2>/dev/null
  for f in b_l141_$rep b_l122_$rep; do python -c "import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'])"; done
done
