# ncu --set full of the f-row kernels: cooperative MFPT solver (1 M states) and the world-model kernel (C4)
python tools/mfpt_probe.py 1048576 > gpurun_out/mfpt_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:mfpt -s 1 -c 1 -o gpurun_out/prof_mfpt -f \
  python tools/mfpt_probe.py 1048576 > gpurun_out/ncu_mfpt.log 2>&1; echo ncu_mfpt=$?
true && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:world_serial -s 3 -c 1 -o gpurun_out/prof_world -f \
  python bench.py --workload c4 --world --steps 1 --warmup 3 --ramp-s 0 --no-cpu-baseline > gpurun_out/ncu_world.log 2>&1; echo ncu_world=$?
