"""Iteration-count probe for the windowed sublattice loop (diagnostic, GPU).

Runs the C5 recipe at a chosen block size and reports, per sweep, the inner-loop iterations, events,
hop evaluations and clamps (host-stepped driver), plus the distribution of the per-vacancy expected event
count R * window and of the smallest barrier -- the straggler domains that set the iteration count.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2604_24091_b200 as akmc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=256)
    ap.add_argument("--model", choices=["mlp", "pair"], default="mlp")
    ap.add_argument("--prec", choices=["fp32", "fp64"], default="fp32")
    ap.add_argument("--sweeps", type=int, default=3)
    ap.add_argument("--lam", type=float, default=0.25)
    ap.add_argument("--residual", type=float, default=0.02)
    ap.add_argument("--no-rates", action="store_true", help="skip the rate-distribution summaries")
    a = ap.parse_args()
    pr = synth.preset("C5")
    cells = (a.cells,) * 3
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.physics_mlp(eps, E0, residual=a.residual, seed=1)
    nvac = max(1, round(pr.n_vac_per_voxel * (a.cells / pr.cells[0]) ** 3))
    if a.cells >= 512:                       # same generator as bench.py (on device, then host copy)
        import torch
        sp = synth.make_lattice_iid(cells, pr.fractions, nvac, seed=pr.seed, device="cuda").cpu().numpy()
    else:
        sp = synth.make_lattice(cells, 1, pr.fractions, nvac, seed=pr.seed)
    win = synth.window_seconds(a.lam, E0[0])
    cfg = akmc.Config(cells=cells, n_voxels=1, barrier_model=akmc.MODEL_MLP if a.model == "mlp" else akmc.MODEL_PAIR,
                      precision=akmc.PREC_FP32 if a.prec == "fp32" else akmc.PREC_FP64,
                      domain_cells=pr.domain, window_s=win, seed=pr.seed)
    sim = akmc.Simulation(cfg, sp, eps, E0, mlp)
    sim.set_profiling(True)

    def rate_stats():
        R, E = sim.rates()
        tot = R.sum(axis=1) * win
        emin = np.where(R > 0, E, np.inf).min(axis=1)
        q = [0.5, 0.9, 0.99, 0.999, 1.0]
        return {"nvac": int(R.shape[0]), "R_win_q": dict(zip(map(str, q), np.quantile(tot, q).round(3).tolist())),
                "n_R_win_gt_10": int((tot > 10).sum()), "n_R_win_gt_100": int((tot > 100).sum()),
                "Emin_q": dict(zip(map(str, [0.0, 0.001, 0.01, 0.5]), np.quantile(emin, [0.0, 0.001, 0.01, 0.5]).round(4).tolist()))}

    print(json.dumps({"cells": a.cells, "nvac": nvac, "window_s": win,
                      "before": None if a.no_rates else rate_stats()}), flush=True)
    for s in range(a.sweeps):
        c = sim.step(1)
        print(json.dumps({"sweep": s, **{k: c[k] for k in ("iterations", "events", "hop_evals", "clamps", "mlp_rows")},
                          "mlp_ms": round(c["mlp_ms"], 2), "wall_ms": round(c["wall_ms"], 2)}), flush=True)
    if not a.no_rates:
        print(json.dumps({"after": rate_stats()}), flush=True)
    sim.close()


if __name__ == "__main__":
    main()
