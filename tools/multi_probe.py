"""Per-sweep timing of the C5 spatial decomposition (torchrun, one rank per GPU): wall time per sweep with the
graph driver and with the host-stepped driver (events around every engine launch), so that engine time and
exchange/other time can be told apart."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402


def main():
    import torch
    import torch.distributed as dist
    import paper_2604_24091_b200 as akmc
    from paper_2604_24091_b200 import dist as D
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=1)
    nid = D.broadcast_nccl_id(rank, device=dev)
    cfg, pr = bench.sim_config("c5", akmc.PREC_FP32, akmc.MODEL_MLP, 0.25, E0, rank, world, nid)
    sp, keep = bench.make_inputs("c5", rank, dev)
    sim = akmc.Simulation(cfg, sp, eps, E0, mlp)
    stream = None
    if os.environ.get("PROBE_TORCH_STREAM"):
        stream = torch.cuda.Stream(device=dev)
        sim.set_stream(stream.cuda_stream)
    cs = None
    if os.environ.get("PROBE_CLOCKS"):
        cs = bench.ClockSampler(local).__enter__()
    out = {"rank": rank, "graph_ms": [], "host_ms": [], "engine_ms": []}
    for _ in range(3):
        sim.step(1)
    for _ in range(4):
        torch.cuda.synchronize()
        t = time.perf_counter()
        sim.step(1)
        torch.cuda.synchronize()
        out["graph_ms"].append(round(1e3 * (time.perf_counter() - t), 2))
    sim.set_profiling(True)
    for _ in range(4):
        c0 = sim.counters()
        t = time.perf_counter()
        sim.step(1)
        torch.cuda.synchronize()
        out["host_ms"].append(round(1e3 * (time.perf_counter() - t), 2))
        out["engine_ms"].append(round(sim.counters()["mlp_ms"] - c0["mlp_ms"], 2))
    if cs:
        cs.__exit__()
    sim.close()
    print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
