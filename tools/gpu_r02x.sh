# world-model time mode: GPU parity tests + bench lines (C4 and C1, --world)
timeout 900 python -m pytest tests/test_gpu_world.py -q -p no:cacheprovider > gpurun_out/pytest_world.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_world.log
for w in c4 c1; do
  timeout 600 python bench.py --workload $w --world > gpurun_out/wl_${w}_world.json 2> gpurun_out/wl_${w}_world.err; echo $w rc=$?
  python -c "import json;d=json.loads(open('gpurun_out/wl_${w}_world.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline']['rows'],d['cpu_baseline']['value'],d['gpu_launches'])"
done
