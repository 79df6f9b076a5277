import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np
import synth, oracle
import paper_2604_24091_b200 as akmc
oracle.build()
eps, E0 = synth.illustrative_pair_params()
pr = synth.preset("C1")
sp = synth.make_lattice(pr.cells, 1, pr.fractions, 1, seed=pr.seed)
cfg = akmc.Config(cells=pr.cells, barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=2605)
ocfg = oracle.Config(cells=cfg.cells, n_voxels=1, T=cfg.temperature_K, nu0=cfg.nu0, kB=cfg.kB, model=0, domain=(0,0,0), window_s=0.0, seed=cfg.seed)
ost = oracle.State.from_species(ocfg, sp)
with akmc.Simulation(cfg, sp, eps, E0) as sim:
    for n in range(1, 40):
        sim.step(1); oracle.run(ocfg, ost, 1, eps, E0)
        gsp, gvac, gclock, gctr = sim.state()
        ok = np.array_equal(gsp, ost.species) and np.array_equal(gvac, ost.vac)
        print(n, ok, gvac, ost.vac, gclock, ost.clock, gctr["events"], ost.counters[0])
        if not ok: break
