# hot-first segment ordering (AKMC_HOT_EVENTS = expected events threshold) A/B at HEAD
for rep in 1 2; do
for he in 0 1 3; do
  AKMC_HOT_EVENTS=$he timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/bh$he$rep.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bh$he$rep.json').read().strip().splitlines()[-1]); print('hot=$he', $rep, d['value'], d['ms_per_step'])"
done
done
