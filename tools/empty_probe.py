"""Diagnostic: sublattice run with no vacancy -- where does the lattice change?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch  # noqa: F401
import synth
import paper_2604_24091_b200 as A

eps, E0 = synth.illustrative_pair_params()
for L, dom in [(16, (8, 8, 8)), (32, (8, 8, 8))]:
    for cu in (0.0, 0.05):
        sp = synth.make_lattice((L, L, L), 1, synth.fe_cu_fractions(cu), 0, seed=1) if cu else np.zeros(2 * L ** 3, np.uint8)
        cfg = A.Config(cells=(L, L, L), barrier_model=A.MODEL_PAIR, precision=A.PREC_FP64, seed=3,
                       domain_cells=dom, window_s=synth.window_seconds(1.0, E0[0]))
        with A.Simulation(cfg, sp, eps, E0) as sim:
            g0, v0, c0, _ = sim.state()
            d0 = np.flatnonzero(g0 != sp)
            c = sim.step(3)
            g1, v1, c1, k1 = sim.state()
            d1 = np.flatnonzero(g1 != sp)
        print(f"L={L} cu={cu}: after init diff={d0.size} {d0[:8]} vals={g0[d0[:8]]}; after step status={c['status']} "
              f"diff={d1.size} {d1[:8]} vals={g1[d1[:8]]} vac={v1.size} clock={c1} events={k1['events']}", flush=True)
