import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, synth, paper_2604_24091_b200 as akmc
eps, E0 = synth.illustrative_pair_params()
mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=1)
sp = synth.make_lattice((64, 64, 64), 8, synth.a508_atomic_fractions(), 10, seed=1)
cfg = akmc.Config(cells=(64, 64, 64), n_voxels=8, barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32)
with akmc.Simulation(cfg, sp, eps, E0, mlp) as sim:
    sim.set_voxel_temperatures(synth.voxel_temperatures(8, seed=7))
    sim.run_until(1e-6)                     # every voxel to 1 microsecond of physical time
    species, vac_sites, clocks, counters = sim.state()
print("quickstart ok", counters["events"], float(clocks.min()))
