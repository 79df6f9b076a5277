"""Time the bulk evaluator (akmc_rates on every vacancy of a C5 block) -- for ncu / A-B runs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    import synth
    import paper_2604_24091_b200 as akmc
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=1)
    cfg, pr = bench.sim_config("c5", akmc.PREC_FP32, akmc.MODEL_MLP, 0.25, E0)
    sp, keep = bench.make_inputs("c5", 0, torch.device("cuda", 0))
    with akmc.Simulation(cfg, sp, eps, E0, mlp) as sim:
        sim.set_profiling(True)
        for r in range(reps):
            c0 = sim.counters()
            sim.rates()
            c1 = sim.counters()
            print(f"rep {r}: {c1['mlp_ms'] - c0['mlp_ms']:.4f} ms for {sim.n_vac} rows", flush=True)


if __name__ == "__main__":
    main()
