# engine gather rows in flight per warp: 8 (default) vs 12 vs 16 (A/B, same box)
for rep in 1 2; do
for v in "" _g12 _g16; do
  if [ -n "$v" ]; then export AKMC_LIB=paper_2604_24091_b200/lib/libakmc$v.so; else unset AKMC_LIB; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/bg$v$rep.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bg$v$rep.json').read().strip().splitlines()[-1]); print('g$v', $rep, d['value'], d['ms_per_step'])"
done
done
