"""Diagnostics: per-phase cycle breakdown of mlp_tc_kernel (AKMC_PHASE_TIMING=1) on explicit windows
and on a C5 sweep.  Not part of the product path."""
import os, sys, time
os.environ["AKMC_PHASE_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2604_24091_b200 as akmc, synth
eps, E0 = synth.illustrative_pair_params()
mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=1)
for n in (128, 148 * 128, 4 * 148 * 128):
    w = synth.random_windows(n, seed=1, solute=0.03, vac=0.001)
    cfg = akmc.Config(cells=(8, 8, 8), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32)
    sim = akmc.Simulation(cfg, np.zeros(1024, np.uint8), mlp=mlp)
    sim.set_profiling(True)
    for _ in range(3):
        sim.eval_windows(w, akmc.PREC_FP32)
    _, _, _, c = sim.state(species=False)
    print(f"n={n}: eval kernel {c['mlp_ms']/c['mlp_launches']*1e3:.1f} us/launch", flush=True)
    sim.close()
