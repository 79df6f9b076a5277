"""compute-sanitizer target: FP32 evaluator on a small window batch and a short FP32 sublattice run."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2604_24091_b200 as akmc  # noqa: E402

eps, E0 = synth.illustrative_pair_params()
mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=4)
w = synth.random_windows(int(sys.argv[1]) if len(sys.argv) > 1 else 127, seed=5)
cfg = akmc.Config(cells=(8, 8, 8), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32)
with akmc.Simulation(cfg, np.zeros(2 * 8 ** 3, np.uint8), eps, E0, mlp) as sim:
    e32 = sim.eval_windows(w, akmc.PREC_FP32)
    e64 = sim.eval_windows(w, akmc.PREC_FP64)
print("eval max |dE|", float(np.max(np.abs(e32 - e64))))
L = 24
sp = synth.make_lattice((L, L, L), 1, synth.a508_atomic_fractions(), 40, seed=42)
cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32, seed=19,
                  domain_cells=(6, 6, 6), window_s=synth.window_seconds(1.0, E0[0]))
with akmc.Simulation(cfg, sp, eps, E0, mlp) as sim:
    c = sim.step(3)
print("sublattice events", c["events"])
