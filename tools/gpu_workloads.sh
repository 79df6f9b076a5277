# one GPU round-trip: build, then bench lines for every workload config (serial: --events per step)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for w in "c5" "c1" "c2" "c3" "c4" "c4 --voxel-T" "c5 --lam 1.0"; do
  n=$(echo $w | tr ' ' '_' | tr -d '-')
  timeout 400 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$n.json 2> gpurun_out/bench_$n.err; echo "$w rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/bench_$n.json'));print('$w', d['value'], d['ms_per_step'], d['events_per_s'], d['sim_seconds_per_wall_second'], d['roofline']['frac'], d['e2e']['value'])" 2>&1 | tail -1
done
