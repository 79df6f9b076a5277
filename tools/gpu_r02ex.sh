# det_exp scaling by a constructed power of two (ldexp's bits): parity suite + A/B timings (bulk evaluator, bench)
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "not multi" > gpurun_out/pytest_ex.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_ex.log
for rep in 1 2; do
  timeout 300 python tools/bulk_probe.py 8 2>&1 | grep rep | tail -2 | sed "s/^/new $rep /"
  AKMC_LIB=paper_2604_24091_b200/lib/libakmc_ldexp.so timeout 300 python tools/bulk_probe.py 8 2>&1 | grep rep | tail -2 | sed "s/^/old $rep /"
  timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/b_ex_$rep.json 2>/dev/null
  AKMC_LIB=paper_2604_24091_b200/lib/libakmc_ldexp.so timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/b_ld_$rep.json 2>/dev/null
  for f in b_ex_$rep b_ld_$rep; do python -c "import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'])"; done
done
