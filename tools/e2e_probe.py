"""Where the end-to-end time of bench.py's e2e leg goes (C5 block on one GPU): akmc_init from a pinned host
lattice, K x (akmc_step + counters), final lattice readback; host wall clock per part."""
import ctypes
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402


def main():
    import torch
    import paper_2604_24091_b200 as akmc
    dev = torch.device("cuda", 0)
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=1)
    cfg, pr = bench.sim_config("c5", akmc.PREC_FP32, akmc.MODEL_MLP, 0.25, E0)
    sp_host, keep = bench.make_inputs("c5", 0, dev)
    torch.cuda.synchronize()
    out = {}
    buf = torch.empty(sp_host.size, dtype=torch.uint8, pin_memory=True).numpy()
    for rep in range(2):
        t0 = time.perf_counter()
        sim = akmc.Simulation(cfg, sp_host, eps, E0, mlp)
        t1 = time.perf_counter()
        steps = []
        for _ in range(5):
            a = time.perf_counter()
            sim.step(1)
            sim.counters()
            steps.append(time.perf_counter() - a)
        t2 = time.perf_counter()
        vac = np.empty(max(sim.n_vac, 1), dtype=np.int64)
        n = ctypes.c_int64(vac.size)
        sim.lib.akmc_state(sim.h, ctypes.c_void_p(buf.ctypes.data), ctypes.c_void_p(vac.ctypes.data), ctypes.byref(n),
                           None, None)
        t3 = time.perf_counter()
        sim.close()
        t4 = time.perf_counter()
        out[f"rep{rep}"] = {"init_s": t1 - t0, "steps_s": [round(x, 4) for x in steps], "readback_s": t3 - t2,
                            "close_s": t4 - t3}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
