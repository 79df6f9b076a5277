# round-2 evidence on one B200: GPU suite, smoke, bench lines (default + reference arm + every workload), launch
# list of the bench command, ncu --set full of one engine launch and one bulk-evaluator launch
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err; echo ref=$?
for w in "c1" "c2" "c3" "c4" "c4 --voxel-T" "c5 --lam 1.0"; do
  n=$(echo $w | tr ' ' '_' | tr -d '-')
  timeout 400 python bench.py --workload $w --no-cpu-baseline > gpurun_out/wl_$n.json 2> gpurun_out/wl_$n.err; echo "$w rc=$?"
done
python bench.py --steps 2 --warmup 3 --ramp-s 0 --no-cpu-baseline > gpurun_out/plain2.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 2 --warmup 3 --ramp-s 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
python tools/iter_probe.py --cells 1024 --sweeps 2 --no-rates > gpurun_out/plain1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:engine_kernel -s 12 -c 1 -o gpurun_out/prof_engine_final -f \
  python tools/iter_probe.py --cells 1024 --sweeps 2 --no-rates > gpurun_out/ncu_full.log 2>&1; echo ncu_engine=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bulk_eval -s 2 -c 1 -o gpurun_out/prof_bulk_final -f \
  python tools/bulk_probe.py 3 > gpurun_out/ncu_bulk.log 2>&1; echo ncu_bulk=$?
tail -3 gpurun_out/pytest_gpu_final.log; tail -1 gpurun_out/smoke.log
python -c "import json; d=json.loads(open('gpurun_out/bench_final.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['evaluator_bulk']['executed_frac'], d['e2e']['value'], d['clocks'])"
