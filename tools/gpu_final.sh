# round-end round trip: GPU tests, smoke, C4 A/B of the serial clock cache, default bench, ncu launch list + full capture
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
L=paper_2604_24091_b200/lib
for rep in 1 2; do for v in libakmc v_noclk; do
  AKMC_LIB=$L/$v.so timeout 300 python bench.py --workload c4 --no-cpu-baseline --ramp-s 0.5 > gpurun_out/ab_c4_${v}_$rep.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_c4_${v}_$rep.json'));print('$v', $rep, round(d['ms_per_step'],4), d['value'])"
done; done
timeout 400 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['clocks'],d['e2e']['value'],d['cpu_baseline']['value'])"
python bench.py --steps 2 --warmup 3 --ramp-s 0 --no-cpu-baseline > gpurun_out/plain2.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --ramp-s 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
python tools/iter_probe.py --cells 1024 --sweeps 2 --no-rates > gpurun_out/plain1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:engine_kernel -s 12 -c 1 -o gpurun_out/prof_engine \
  python tools/iter_probe.py --cells 1024 --sweeps 2 --no-rates > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
