# hot-first segment order: correctness + A/B by AKMC_HOT_EVENTS (0 = off) on one box
timeout 900 python -m pytest tests -m gpu -x -q -k "sublattice or engine or fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for rep in 1 2 3; do
  for he in 0 1 0.5 2; do
    AKMC_HOT_EVENTS=$he timeout 300 python tools/iter_probe.py --cells 1024 --sweeps 5 --no-rates > gpurun_out/hot_${he}_$rep.log 2>&1
    python - <<PY
import json
rows=[json.loads(l) for l in open("gpurun_out/hot_${he}_$rep.log") if l.startswith('{"sweep"')]
print("he=$he rep=$rep", [round(r["wall_ms"],3) for r in rows], [r["events"] for r in rows])
PY
  done
done
for he in 0 1; do
  AKMC_HOT_EVENTS=$he AKMC_PHASE_TIMING=1 timeout 300 python tools/iter_probe.py --cells 1024 --sweeps 4 --no-rates > gpurun_out/hot_t$he.log 2>&1
  echo he=$he; grep -E "iterations/CTA" gpurun_out/hot_t$he.log | head -2
done
