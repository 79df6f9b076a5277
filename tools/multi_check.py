"""Multi-GPU spatial decomposition check (C5 path): run the same global problem on
`world` ranks (halo deltas between phases) and on one rank, and compare the final global lattices,
vacancy lists, clocks and event counts bit for bit (GPU-count invariance); optionally also against the
FP64 CPU oracle.  Launch:  torchrun --nproc-per-node N tools/multi_check.py --grid gx gy gz ..."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as tdist

    import paper_2604_24091_b200 as akmc
    import synth
    from paper_2604_24091_b200 import dist as D

    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, nargs=3, default=[2, 1, 1])
    ap.add_argument("--cells", type=int, nargs=3, default=[16, 16, 16])
    ap.add_argument("--sweeps", type=int, default=6)
    ap.add_argument("--nvac", type=int, default=40)
    ap.add_argument("--domain", type=int, nargs=3, default=[8, 8, 8])
    ap.add_argument("--lam", type=float, default=1.0)
    ap.add_argument("--model", default="pair", choices=["pair", "mlp"])
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--debug", action="store_true")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    grid, block = tuple(a.grid), tuple(a.cells)
    assert grid[0] * grid[1] * grid[2] == world
    G = tuple(b * g for b, g in zip(block, grid))
    glob = synth.make_lattice(G, 1, synth.fe_cu_fractions(0.05), a.nvac, seed=77)
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=3) if a.model == "mlp" else None
    model = akmc.MODEL_MLP if a.model == "mlp" else akmc.MODEL_PAIR
    prec = akmc.PREC_FP32 if a.precision == "fp32" else akmc.PREC_FP64
    win = synth.window_seconds(a.lam, E0[0])
    nid = D.broadcast_nccl_id(rank, device=torch.device("cuda", local))
    cfg = akmc.Config(cells=block, barrier_model=model, precision=prec, domain_cells=tuple(a.domain), window_s=win, seed=5,
                      gpu_grid=grid, rank=rank, world=world, nccl_id=nid)
    sim = akmc.Simulation(cfg, D.block_of(glob, block, grid, rank), eps, E0, mlp)
    if a.debug:
        # lockstep with a single-rank reference; after every sweep each rank's extended block (halo
        # included) must equal the reference global lattice around its block (periodic images)
        ref = akmc.Simulation(akmc.Config(cells=G, barrier_model=model, precision=prec, domain_cells=tuple(a.domain),
                                          window_s=win, seed=5), glob, eps, E0, mlp)
        cx, cy, cz = D.rank_coords(rank, grid)
        O = (cx * block[0], cy * block[1], cz * block[2])
        for sw in range(a.sweeps + 1):
            rsp, _, _, _ = ref.state()
            g4 = rsp.reshape(G[2], G[1], G[0], 2)
            ext = sim.debug_extended().reshape(block[2] + 4, block[1] + 4, block[0] + 4, 2)
            zz = (np.arange(-2, block[2] + 2) + O[2]) % G[2]
            yy = (np.arange(-2, block[1] + 2) + O[1]) % G[1]
            xx = (np.arange(-2, block[0] + 2) + O[0]) % G[0]
            want = g4[zz][:, yy][:, :, xx]
            bad = np.argwhere(ext != want)
            print(f"[rank {rank}] sweep {sw}: {len(bad)} mismatching sites"
                  + (f", first (z,y,x,b) local {tuple(int(t) - (2 if i < 3 else 0) for i, t in enumerate(bad[0]))}"
                     f" got {ext[tuple(bad[0])]} want {want[tuple(bad[0])]}" if len(bad) else ""), flush=True)
            flag = torch.tensor([len(bad)], device=torch.device("cuda", local))
            tdist.all_reduce(flag)                      # collective decision: no rank may stop alone
            if int(flag.item()) or sw == a.sweeps:
                break
            sim.step(1)
            ref.step(1)
        ref.close()
        c = {"events": 0, "hop_evals": 0}
    else:
        c = sim.step(a.sweeps)
    sp, _, clock, _ = sim.state()
    gid, site = sim.vacancies()
    xs = sim.exchange_stats()
    sim.close()
    parts = [None] * world
    tdist.all_gather_object(parts, (sp, gid, site, float(clock[0]), int(c["events"]), int(c["hop_evals"]), xs))
    result = {}
    if rank == 0:
        gsp = D.assemble([p[0] for p in parts], block, grid)
        gids = np.concatenate([p[1] for p in parts])
        sites = np.concatenate([p[2] for p in parts])
        order = np.argsort(gids)
        events = sum(p[4] for p in parts)
        hop = sum(p[5] for p in parts)
        ref_cfg = akmc.Config(cells=G, barrier_model=model, precision=prec, domain_cells=tuple(a.domain), window_s=win, seed=5)
        ref = akmc.Simulation(ref_cfg, glob, eps, E0, mlp)
        rc = ref.step(a.sweeps)
        rsp, rvac, rclock, _ = ref.state()
        ref.close()
        result = {"world": world, "grid": grid, "events": events, "ref_events": int(rc["events"]),
                  "exchange": os.environ.get("AKMC_EXCHANGE", "p2p"),
                  "messages_per_phase": [p[6]["messages"] / max(p[6]["exchanges"], 1) for p in parts],
                  "hop_evals": hop, "ref_hop_evals": int(rc["hop_evals"]),
                  "species_equal": bool(np.array_equal(gsp, rsp)),
                  "vacancies_equal": bool(np.array_equal(gids[order], np.arange(gids.size))) and
                                     bool(np.array_equal(sites[order], rvac)),
                  "clock_equal": all(p[3] == float(rclock[0]) for p in parts)}
        if a.oracle:
            import oracle
            oc = oracle.Config(cells=G, model=model, domain=tuple(a.domain), window_s=win, seed=5)
            st = oracle.State.from_species(oc, glob)
            oracle.run(oc, st, a.sweeps, eps, E0, mlp)
            result["oracle_species_equal"] = bool(np.array_equal(gsp, st.species))
            result["oracle_vacancies_equal"] = bool(np.array_equal(sites[order], st.vac))
        result["ok"] = all(v for k, v in result.items() if k.endswith("_equal")) and result["events"] == result["ref_events"]
        print(json.dumps(result), flush=True)
        if a.out:
            with open(a.out, "w") as f:
                json.dump(result, f)
    tdist.barrier()
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
