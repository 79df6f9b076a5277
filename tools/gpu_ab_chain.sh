# memo-hit chain: correctness (GPU parity suite) + A/B timing of chain variants on one box
L=paper_2604_24091_b200/lib
timeout 900 python -m pytest tests -m gpu -x -q -k "sublattice or serial or engine or voxel" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for v in off:v_off all:libakmc n16:v_n16 n4:v_n48; do
  AKMC_LIB=$L/${v#*:}.so AKMC_PHASE_TIMING=1 timeout 300 python tools/iter_probe.py --cells 1024 --sweeps 4 --no-rates > gpurun_out/iter_${v%%:*}.log 2>&1
  echo ${v%%:*}; grep -E "chain|iterations/CTA" gpurun_out/iter_${v%%:*}.log | head -3
done
timeout 900 python tools/ab_probe.py off=$L/v_off.so all=$L/libakmc.so n16=$L/v_n16.so n4=$L/v_n48.so --cells 1024 --sweeps 5 --reps 3 > gpurun_out/ab_chain.log 2>&1
tail -4 gpurun_out/ab_chain.log
