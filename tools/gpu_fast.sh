# FP16 fast mode: GPU tests + C5 bench A/B against the FP32-equivalent mode (same box, alternating)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
grep -E "Error|assert" gpurun_out/pytest_gpu.log | head -5
for rep in 1 2; do for pr in fp32 fast; do
  timeout 300 python bench.py --precision $pr --no-cpu-baseline --ramp-s 0.5 > gpurun_out/fast_${pr}_$rep.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/fast_${pr}_$rep.json'));r=d['roofline'];print('$pr', $rep, round(d['ms_per_step'],4), d['value'], r['evaluator_bulk']['ms'], r['frac'])"
done; done
