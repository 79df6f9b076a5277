"""Dataflow sweep vs phase-synchronous sweep on C5 (1024^3, 214,748 vacancies, FP32 MLP): ms per sweep with CUDA
events (graph mode, as bench.py), plus the bit-identity of the two trajectories after the timed sweeps."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    import synth
    import paper_2604_24091_b200 as akmc
    sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    lam = float(sys.argv[2]) if len(sys.argv) > 2 else 0.25
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=1)
    cfg, pr = bench.sim_config("c5", akmc.PREC_FP32, akmc.MODEL_MLP, lam, E0)
    sp, keep = bench.make_inputs("c5", 0, torch.device("cuda", 0))
    out = {}
    for mode in ("sync", "dataflow"):
        with akmc.Simulation(cfg, sp, eps, E0, mlp) as sim:
            if mode == "dataflow":
                sim.set_dataflow(True)
            stream = torch.cuda.Stream()
            sim.set_stream(stream.cuda_stream)
            sim.step(3)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            c0 = sim.counters()
            e0.record(stream)
            sim.step(sweeps)
            e1.record(stream)
            torch.cuda.synchronize()
            c1 = sim.counters()
            ms = e0.elapsed_time(e1) / sweeps
            st = sim.state()
            out[mode] = st
            print(f"{mode}: {ms:.3f} ms/sweep, {(c1['hop_evals'] - c0['hop_evals']) / (ms * 1e-3 * sweeps):.4e} hop-evals/s, "
                  f"{c1['events'] - c0['events']} events", flush=True)
    same = all(np.array_equal(a, b) for a, b in zip(out["sync"][:3], out["dataflow"][:3]))
    print("trajectories identical:", same, flush=True)


if __name__ == "__main__":
    main()
