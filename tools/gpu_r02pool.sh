# pooled device allocations: single-GPU suite + bench e2e init (AKMC_VERBOSE laps)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "not multi" > gpurun_out/pytest_pool.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_pool.log
for rep in 1 2; do
AKMC_VERBOSE=1 timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/b_pool$rep.json 2> gpurun_out/b_pool$rep.err
grep "akmc init" gpurun_out/b_pool$rep.err | tail -9 | awk '{s+=$(NF-1)} END {print "init laps ms:", s}'
python -c "import json; d=json.loads(open('gpurun_out/b_pool$rep.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['parts'])"
done
