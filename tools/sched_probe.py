"""Dynamic voxel scheduling A/B (Eq. 10): a voxel batch larger than the engine's resident slots with
heterogeneous temperatures, advanced to a common time (akmc_run_until).  Run twice: default (descending W_v) and
AKMC_VOXEL_FIFO=1 (voxel-id order); same trajectories, different makespan."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import synth
    import paper_2604_24091_b200 as akmc
    nvox = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
    L = 8
    eps, E0 = synth.illustrative_pair_params()
    rng = np.random.default_rng(7)
    S = 2 * L ** 3
    sp = np.zeros(nvox * S, dtype=np.uint8)
    base = synth.make_lattice((L, L, L), 1, synth.a508_atomic_fractions(), 2, seed=1)
    for v in range(nvox):
        sp[v * S:(v + 1) * S] = np.roll(base, int(rng.integers(0, S // 2)) * 2)
    T = rng.uniform(520.0, 620.0, size=nvox)            # wide T spread: heterogeneous event rates
    cfg = akmc.Config(cells=(L, L, L), n_voxels=nvox, barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=3)
    t_end = 2.0e-7
    with akmc.Simulation(cfg, sp, eps, E0) as sim:
        sim.set_voxel_temperatures(T)
        sim.run_until(t_end * 0.01)                     # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        c = sim.run_until(t_end)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        _, vac, clock, _ = sim.state(species=False)
    print(f"{'FIFO' if os.environ.get('AKMC_VOXEL_FIFO') else 'W_v priority'}: {nvox} voxels, {c['events']} events, "
          f"{dt * 1e3:.2f} ms, checksum {int(vac.sum())} {float(clock.sum()):.9e}", flush=True)


if __name__ == "__main__":
    main()
