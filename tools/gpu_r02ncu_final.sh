# HEAD: launch list of the bench command and ncu --set full of one engine phase launch (profiles evidence)
python bench.py --steps 2 --warmup 3 --ramp-s 0 --no-cpu-baseline > gpurun_out/plain2.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 2 --warmup 3 --ramp-s 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
python tools/iter_probe.py --cells 1024 --sweeps 2 --no-rates > gpurun_out/plain1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:engine_kernel -s 12 -c 1 -o gpurun_out/prof_engine_final -f \
  python tools/iter_probe.py --cells 1024 --sweeps 2 --no-rates > gpurun_out/ncu_full.log 2>&1; echo ncu_engine=$?
