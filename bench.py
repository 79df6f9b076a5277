#!/usr/bin/env python
"""Benchmark of the B200 AKMC hot path (BASELINE.json metric: vacancy-hop evaluations/sec and
simulated seconds per wall-second at 1/2/4/8 B200).

Default workload = C5: 1024^3 bcc cells per GPU (2.1e9 sites), c_v = 1e-4 (214,748 vacancies),
RPV composition, windowed synchronous sublattice (domains 8^3, lambda = 1/4), barrier network
448-256-256-8 (physics-embedded weights + seeded residual) in the tensor-core FP32-equivalent mode.
A step = one sublattice sweep (8 phases) over the GPU's block.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c5|c4|c3|c2|c1]
  python bench.py --workload c4 --world      (the world-model time mode, on a serial workload)
  python bench.py --workload c1 --replicas 4096   (C1's batched-replica variant for throughput)

N > 1 is launched by torchrun (one rank per GPU).  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "vacancy-hop evaluations/sec"
UNIT = "hop-evals/s"
FLOPS_PER_VAC = 2 * (256 * 256 + 256 * 8) + 64 * 256      # layers 2-3 FLOPs + layer-1 adds
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
# DRAM bytes (read + write) per engine launch from the committed ncu --set full capture (profiles/)
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r02_engine_ncu.json")


def _traffic():
    try:
        return json.load(open(TRAFFIC_FILE)).get("dram_bytes_per_launch")
    except Exception:
        return None


TRAFFIC_PER_LAUNCH = _traffic()
GATHER_BYTES_PER_VAC = 64 + 16      # SURVEY 8(d) algorithmic work per vac: window + vacancy record


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


REPLICAS = None                         # --replicas: serial workloads as a batch of independent replica voxels


def workload(name: str):
    pr = synth.preset(name.upper())
    cells = pr.cells
    nvox = pr.n_voxels
    if name == "c4":
        nvox = 512                      # per GPU (4096 over 8 GPUs)
    if REPLICAS and not pr.domain[0]:
        nvox = REPLICAS                 # (C1 "plus a batched-replica variant for throughput")
    return pr, cells, nvox


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["stdbuf", "-oL", "nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def make_inputs(name: str, rank: int, device):
    """Synthetic inputs (seeded; recipe in DESIGN.md sec. 4).  Returns host species (pinned numpy)."""
    import torch
    pr, cells, nvox = workload(name)
    seed = pr.seed + 1000 * rank
    if name in ("c5", "c3"):
        t = synth.make_lattice_iid(cells, pr.fractions, pr.n_vac_per_voxel, seed=seed, device=device)
        host = torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True)
        host.copy_(t)
        del t
        return host.numpy(), host
    sp = synth.make_lattice(cells, nvox, pr.fractions, pr.n_vac_per_voxel, seed=seed)
    host = torch.from_numpy(sp).pin_memory()
    return host.numpy(), host


def sim_config(name: str, precision: int, model: int, lam: float, E0, rank: int = 0, world: int = 1, nccl_id=b""):
    """C3/C5 (sublattice) at N > 1: the global lattice is grid_for(N) blocks of `cells`, one per rank, with
    halo deltas between phases over NVLink peer memory; C1/C2/C4 (serial BKL): independent voxels per rank, no collective."""
    import paper_2604_24091_b200 as akmc
    from paper_2604_24091_b200 import dist as D
    pr, cells, nvox = workload(name)
    win = synth.window_seconds(lam, E0[0]) if pr.domain[0] else 0.0
    decomposed = bool(pr.domain[0]) and world > 1
    return akmc.Config(cells=cells, n_voxels=nvox, barrier_model=model, precision=precision,
                       domain_cells=pr.domain, window_s=win, seed=pr.seed,
                       gpu_grid=D.grid_for(world) if decomposed else (1, 1, 1),
                       rank=rank if decomposed else 0, world=world if decomposed else 1,
                       nccl_id=nccl_id if decomposed else b""), pr


def cpu_baseline(name: str, steps: int, lam: float, seconds_target: float = 15.0, world: bool = False):
    """The oracle as it stands (single thread, FP64 MLP) on a bounded sample of the workload."""
    import oracle
    oracle.build()
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=1)
    pr, cells, nvox = workload(name)
    if world:
        # world-model mode: one voxel of the serial recipe, orc_run_world events
        pol, tnet, H, tau = world_nets(E0)
        sp = synth.make_lattice(cells, 1, pr.fractions, pr.n_vac_per_voxel, seed=pr.seed)
        cfg = oracle.Config(cells=cells, model=1, seed=pr.seed)
        st = oracle.State.from_species(cfg, sp)
        t0 = time.perf_counter()
        done = 0
        while True:
            oracle.run_world(cfg, st, 1, eps, E0, pol, tnet, H, tau)
            done += 1
            el = time.perf_counter() - t0
            if el >= seconds_target or done >= max(steps, 1) * 1000:
                break
        hop = int(st.counters[1])
        return {"value": hop / el, "unit": UNIT, "cores": 1, "kind": "oracle", "steps": done,
                "sample": f"one {cells[0]}^3 voxel of {name.upper()} ({pr.n_vac_per_voxel} V), world-model events "
                          f"(orc_run_world, FP64); {done} step(s), {hop} hop evals in {el:.1f} s", **cpu_info()}, st, el
    if pr.domain[0]:
        # sample: a 256^3-cell block of the same recipe (same c_v, domains, lambda), whole sweeps
        sc = (256, 256, 256)
        nvac = max(1, int(round(pr.n_vac_per_voxel * (256 ** 3) / (cells[0] * cells[1] * cells[2]))))
        import torch
        sp = synth.make_lattice_iid(sc, pr.fractions, nvac, seed=pr.seed, device="cpu").numpy()
        cfg = oracle.Config(cells=sc, model=1, domain=pr.domain, window_s=synth.window_seconds(lam, E0[0]),
                            seed=pr.seed)
        sample = f"{sc[0]}^3-cell block of the {name.upper()} recipe ({nvac} V), whole sublattice sweeps, FP64 MLP"
    else:
        sc = cells
        sp = synth.make_lattice(sc, 1, pr.fractions, pr.n_vac_per_voxel, seed=pr.seed)
        cfg = oracle.Config(cells=sc, model=1, seed=pr.seed)
        sample = f"one {sc[0]}^3 voxel of {name.upper()} ({pr.n_vac_per_voxel} V), serial BKL events, FP64 MLP"
    st = oracle.State.from_species(cfg, sp)
    t0 = time.perf_counter()
    done = 0
    while True:
        oracle.run(cfg, st, 1, None, None, mlp)
        done += 1
        el = time.perf_counter() - t0
        if el >= seconds_target or done >= max(steps, 1) * 1000:
            break
    hop = int(st.counters[1])
    return {"value": hop / el, "unit": UNIT, "cores": 1, "kind": "oracle", "steps": done,
            "sample": f"{sample}; {done} step(s), {hop} hop evals in {el:.1f} s", **cpu_info()}, st, el


WORLD_H = 32
FP64_PEAK_TFLOPS = 45.0     # B200 FP64 (blackwell_cuda_programming.md: "B200's 45"); the world mode's FP64 ceiling


def world_nets(E0, T=563.0):
    """World-model mode inputs (reading W2): policy logits z = -E/kT of the physics network (Eq. 2's law is then
    the BKL law), a seeded Poisson-time net of width WORLD_H, tau_act = 1."""
    eps, _ = synth.illustrative_pair_params()
    phys = synth.physics_mlp(eps, E0, residual=0.02, seed=1)
    return synth.policy_mlp(phys, 8.617333262e-5 * T), synth.poisson_net(7, H=WORLD_H), WORLD_H, 1.0


def cpu_info() -> dict:
    """Host CPU facts for the baseline lines (report nproc and the CPU model)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count() or 1
    return {"nproc": usable, "cpu_count": os.cpu_count(), "cpu_model": model}


def _oracle_worker(job):
    """One all-cores worker: the unmodified oracle on its own seeded sample for ~`secs` seconds."""
    name, lam, secs, seed = job
    import oracle
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=1)
    pr, cells, nvox = workload(name)
    if pr.domain[0]:
        import torch
        torch.set_num_threads(1)                        # one core per worker
        sc = (128, 128, 128)
        nvac = max(1, int(round(pr.n_vac_per_voxel * (128 ** 3) / (cells[0] * cells[1] * cells[2]))))
        sp = synth.make_lattice_iid(sc, pr.fractions, nvac, seed=seed, device="cpu").numpy()
        cfg = oracle.Config(cells=sc, model=1, domain=pr.domain, window_s=synth.window_seconds(lam, E0[0]), seed=seed)
    else:
        sp = synth.make_lattice(cells, 1, pr.fractions, pr.n_vac_per_voxel, seed=seed)
        cfg = oracle.Config(cells=cells, model=1, seed=seed)
    st = oracle.State.from_species(cfg, sp)
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < secs:
        oracle.run(cfg, st, 1, None, None, mlp)
    return int(st.counters[1]), time.perf_counter() - t0


def cpu_baseline_all_cores(name: str, lam: float, secs: float = 8.0) -> dict:
    """The same oracle, one independent seeded sample per host core (domains / voxels are independent units of
    the method), summed hop-evals over the slowest worker's time."""
    import multiprocessing as mp
    import oracle
    oracle.build()
    n = cpu_info()["nproc"]
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(n) as pool:          # spawn: the parent holds a CUDA context
        res = pool.map(_oracle_worker, [(name, lam, secs, 9000 + i) for i in range(n)])
    el = max(r[1] for r in res)
    hop = sum(r[0] for r in res)
    pr, _, _ = workload(name)
    unit = ("128^3-cell blocks of the recipe, whole sublattice sweeps" if pr.domain[0]
            else "voxels of the recipe, serial BKL events")
    return {"value": hop / el, "unit": UNIT, "cores": n, "kind": "oracle",
            "sample": f"{n} workers x one seeded {unit}, FP64 MLP, ~{secs:.0f} s each; {hop} hop evals "
                      f"(wall {time.perf_counter() - t0:.1f} s incl. setup)"}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    t_all = time.perf_counter()
    cb, st, el = cpu_baseline(args.workload, args.steps, args.lam, seconds_target=max(10.0, 4.0 * args.steps),
                              world=args.world)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / max(cb["steps"], 1),
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload.upper(), "impl": "CPU FP64 oracle (oracle/akmc_oracle.c)",
                       "step": "one oracle step of the bounded sample named in cpu_baseline.sample"},
            "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t_all}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2604_24091_b200 as akmc
    from paper_2604_24091_b200 import build as akbuild

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        akbuild.build()
    if world > 1:
        dist.barrier()
    prec = {"fp32": akmc.PREC_FP32, "fp64": akmc.PREC_FP64, "fast": akmc.PREC_FP16_FAST}[args.precision]
    model = akmc.MODEL_MLP if args.model == "mlp" else akmc.MODEL_PAIR
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=1)
    wnets = None
    if args.world:
        if workload(args.workload)[0].domain[0]:
            raise SystemExit("--world: serial workloads only (c1, c2, c4)")
        prec, model = akmc.PREC_FP64, akmc.MODEL_MLP       # the world mode is FP64 (bit-exact with orc_run_world)
        wnets = world_nets(E0)
        mlp = wnets[0]
    from paper_2604_24091_b200 import dist as D
    nid = D.broadcast_nccl_id(rank, device=dev) if world > 1 else b""
    cfg, pr = sim_config(args.workload, prec, model, args.lam, E0, rank, world, nid)
    sp_host, sp_keep = make_inputs(args.workload, rank, dev)
    sites = sp_host.size

    # one step = one sweep of 8 phases (sublattice) or `--events` BKL events of every voxel in one engine
    # launch (serial C1/C2/C4: the per-launch setup is amortised as in a production run of 1e4-1e5 events)
    nstep = 1 if pr.domain[0] else max(1, args.events)
    stream = torch.cuda.Stream(device=dev)
    # ---------------- device-resident timing ("value"): production path (per-sweep CUDA graph)
    sim = akmc.Simulation(cfg, sp_host, eps, E0, mlp)
    if wnets:
        sim.set_world_model(wnets[1], wnets[2], wnets[3])
    vT = None
    if args.voxel_T:
        # C4 variant: per-voxel T uniform in 558-577 K, distinct per rank
        vT = synth.voxel_temperatures(cfg.n_voxels, seed=pr.seed + 1000 * rank + 7)
        sim.set_voxel_temperatures(vT)
    sim.set_stream(stream.cuda_stream)
    cs = ClockSampler(local).__enter__()
    t_ramp = time.perf_counter()                      # untimed clock ramp before the warm-up steps
    flag = torch.ones(1, dtype=torch.int32, device=dev)
    while True:
        # every rank must run the same number of steps (each sweep exchanges halo deltas with the peers):
        # rank 0's clock decides when the ramp ends
        flag.fill_(1 if time.perf_counter() - t_ramp < args.ramp_s else 0)
        if world > 1:
            dist.broadcast(flag, src=0)
        if not int(flag.item()):
            break
        sim.step(nstep)
    for _ in range(args.warmup):
        sim.step(nstep)
    torch.cuda.synchronize()
    _, _, clock0, tot0 = sim.state(species=False)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        sim.step(nstep)
    e1.record(stream)
    torch.cuda.synchronize()
    cs.__exit__()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    _, _, clock1, tot1 = sim.state(species=False)
    hop = tot1["hop_evals"] - tot0["hop_evals"]
    events = tot1["events"] - tot0["events"]
    launches = tot1["kernel_launches"] - tot0["kernel_launches"]
    sim_s = float(np.mean(clock1 - clock0))
    # ---------------- instrumented pass (untimed for `value`): CUDA events around every barrier-kernel
    # launch on the launching stream, same workload continued for K more sweeps
    sim.set_profiling(True)
    _, _, _, p0 = sim.state(species=False)
    pe0 = torch.cuda.Event(enable_timing=True)
    pe1 = torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    for _ in range(args.steps):
        sim.step(nstep)
    pe1.record(stream)
    torch.cuda.synchronize()
    _, _, _, p1 = sim.state(species=False)
    prof_ms = pe0.elapsed_time(pe1)
    mlp_ms = p1["mlp_ms"] - p0["mlp_ms"]
    mlp_launch = p1["mlp_launches"] - p0["mlp_launches"]
    mlp_rows = p1["mlp_rows"] - p0["mlp_rows"]
    logical_rows = (p1["hop_evals"] - p0["hop_evals"]) // 8     # the method's vacancy evaluations (R4)
    bulk = None
    if model and prec != akmc.PREC_FP64:
        _, _, _, q0 = sim.state(species=False)
        sim.rates()
        _, _, _, q1 = sim.state(species=False)
        bulk = {"rows": int(sim.n_vac), "ms": q1["mlp_ms"] - q0["mlp_ms"]}
    sim.close()

    # ---------------- end to end through the C-ABI with host buffers (init H2D + steps + state D2H)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    out = torch.empty(sites, dtype=torch.uint8, pin_memory=True).numpy()   # the caller's pinned result buffer
    if cfg.world > 1:                                   # a fresh communicator for the second handle
        cfg.nccl_id = D.broadcast_nccl_id(rank, device=dev)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    sim2 = akmc.Simulation(cfg, sp_host, eps, E0, mlp)
    if wnets:
        sim2.set_world_model(wnets[1], wnets[2], wnets[3])
    if vT is not None:
        sim2.set_voxel_temperatures(vT)
    t_init = time.perf_counter() - t0
    hop_e2e = 0
    for _ in range(args.steps):
        c = sim2.step(nstep)
        hop_e2e += c["hop_evals"]
        sim2.counters()                                  # the step's result: counters read back to the host
    t_steps = time.perf_counter() - t0 - t_init
    import ctypes
    vac = np.empty(max(sim2.n_vac, 1), dtype=np.int64)
    n = ctypes.c_int64(vac.size)
    sim2.lib.akmc_state(sim2.h, ctypes.c_void_p(out.ctypes.data), ctypes.c_void_p(vac.ctypes.data), ctypes.byref(n),
                        None, None)
    t_e2e = time.perf_counter() - t0
    e2e_parts = {"init_s": t_init, "steps_s": t_steps, "readback_s": t_e2e - t_init - t_steps}
    sim2.close()

    vals = torch.tensor([ms, float(hop), float(events), sim_s, t_e2e, float(hop_e2e), float(launches), mlp_ms,
                         float(mlp_rows), float(mlp_launch)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = vals.clone(); dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vals.clone(); dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    else:
        mx = sm = vals
    ms_max = float(mx[0])
    hop_all = float(sm[1])
    value = hop_all / (ms_max / 1e3)
    e2e_value = float(sm[5]) / float(mx[4])

    line = None
    if rank == 0:
        peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
        tc_peak = peaks.get("bf16_tflops_sustained", 1400.0) * 0.5
        mlp_s = mlp_ms / 1e3 if mlp_ms > 0 else float("nan")
        # SURVEY 8 unit "vac" = one active vacancy in one inner iteration (8 hop evaluations, the metric's unit):
        # achieved = vacs the engine launches processed x 151,552 algorithmic FLOPs / engine time.  The exact memo
        # (R7) serves part of them without running the network; the executed-row rate is reported beside it.
        achieved = (logical_rows * FLOPS_PER_VAC) / mlp_s / 1e12 if mlp_ms > 0 else None
        executed = (mlp_rows * FLOPS_PER_VAC) / mlp_s / 1e12 if mlp_ms > 0 else None
        roof = {"bound": "latency",
                "ceiling": "tensor (FP32-class): the roofline the contraction would hit if the dependent event chain "
                           "did not bound the engine first",
                "kernel": "engine_kernel (phase engine: gather + memo + layer 1 on CUDA cores + tcgen05 layers 2-3 + "
                          "rates + BKL select/apply, one persistent cluster launch per phase)",
                "achieved": achieved, "peak": tc_peak, "unit": "TFLOP/s",
                "frac": (achieved / tc_peak) if achieved else None, "traffic": TRAFFIC_PER_LAUNCH,
                "peak_note": "FP32-class tensor peak = measured bf16 sustained x 1/2 (TF32:BF16 nominal ratio)",
                "algorithmic_flops_per_vac": FLOPS_PER_VAC,
                "work": "active vacancy-iterations processed (SURVEY 8 unit 'vac' = hop_evals / 8) x algorithmic FLOPs "
                        "per vac",
                "launches": int(mlp_launch), "vacs": int(logical_rows),
                "kernel_ms": mlp_ms, "avg_launch_us": 1e3 * mlp_ms / max(mlp_launch, 1),
                "share_of_step": (mlp_ms / ms) if ms > 0 else None,
                "latency_bound": "the phase engine runs each domain's event chain to the window end; its time is "
                                 "set by dependent event latency, not by tensor throughput (DESIGN.md sec. 8)",
                "timing": "CUDA events around each engine launch in an instrumented pass of K further sweeps "
                          f"(host-stepped, {prof_ms:.2f} ms); share = kernel ms / graph-mode step ms"}
        if mlp_ms > 0:
            # north star: achieved HBM GB/s of the gather/encode/select work, beside the tensor roofline.
            # Algorithmic bytes per vac: 64 B window + 16 B vacancy record; measured DRAM bytes per
            # launch from the committed ncu capture (cold caches) over the warm average launch time.
            hbm_peak = peaks.get("hbm_gbs", 6552.0)
            alg_gbs = logical_rows * GATHER_BYTES_PER_VAC / mlp_s / 1e9
            dram_gbs = (TRAFFIC_PER_LAUNCH / (1e-3 * mlp_ms / max(mlp_launch, 1)) / 1e9) if TRAFFIC_PER_LAUNCH else None
            roof["hbm"] = {"achieved": alg_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": alg_gbs / hbm_peak,
                           "bytes_per_vac": GATHER_BYTES_PER_VAC,
                           "dram_achieved": dram_gbs, "dram_frac": (dram_gbs / hbm_peak) if dram_gbs else None,
                           "what": "gather/encode/select bytes (64 B window + 16 B record per vac) / engine time; "
                                   "dram_achieved = ncu DRAM bytes per launch / warm average launch time"}
        if wnets and mlp_ms > 0:
            w_ach = mlp_rows * FLOPS_PER_VAC / mlp_s / 1e12
            roof = {"bound": "latency", "ceiling": "fp64 (CUDA cores)",
                    "kernel": "world_serial_kernel (akmc_world.cu: one CTA per voxel; dirty rows through the FP64 "
                              "network, policy softmax tree, Philox draw, Eq. 7 clock)",
                    "achieved": w_ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": w_ach / FP64_PEAK_TFLOPS,
                    "traffic": None, "algorithmic_flops_per_vac": FLOPS_PER_VAC, "rows": int(mlp_rows),
                    "launches": int(mlp_launch), "kernel_ms": mlp_ms,
                    "share_of_step": (mlp_ms / ms) if ms > 0 else None,
                    "peak_note": "B200 FP64 45 TFLOP/s (guide figure, not measured)",
                    "latency_bound": "each voxel's event chain is serial (one event at a time, S:195-203); a row's "
                                     "FP64 layers run as 256-thread dot products inside the voxel's CTA",
                    "work": "network rows actually evaluated (windows that changed) x 151,552 FLOPs / kernel time"}
        if executed and not wnets:
            roof["executed"] = {"rows": int(mlp_rows), "achieved": executed, "frac": executed / tc_peak,
                                "what": "network rows actually run (memo misses) x algorithmic FLOPs / engine time; the "
                                        f"memo served {1.0 - mlp_rows / max(logical_rows, 1):.0%} of the vacs"}
        if bulk is not None:
            b_ach = bulk["rows"] * FLOPS_PER_VAC / (bulk["ms"] / 1e3) / 1e12
            fp16_sus = peaks.get("bf16_tflops_sustained", 1400.0)       # fp16 dense rate = bf16 rate (guide)
            passes = 1 if prec == akmc.PREC_FP16_FAST else 3
            b_exe = bulk["rows"] * passes * 2 * 256 * 256 / (bulk["ms"] / 1e3) / 1e12
            roof["evaluator_bulk"] = {"rows": bulk["rows"], "ms": bulk["ms"], "achieved": b_ach, "peak": tc_peak,
                                      "frac": b_ach / tc_peak, "unit": "TFLOP/s",
                                      "executed_tensor_tflops": b_exe, "executed_peak": fp16_sus,
                                      "executed_frac": b_exe / fp16_sus,
                                      "kernel": "bulk_eval_kernel (akmc_bulk.cu): persistent, warp-specialised "
                                                "(W2 TMA ring, single-thread tcgen05 issuer, FP64 layer-1 producers, "
                                                "TMEM epilogue with FP64 layer 3)",
                                      "what": "akmc_rates on every vacancy of the block at once, CUDA events around the "
                                              "launch; achieved = algorithmic FP32-class FLOPs (151,552 per row) vs the "
                                              "FP32-class peak; executed = the 3 fp16 passes of layer 2 actually run on "
                                              "the tensor cores vs the measured sustained fp16/bf16 peak"}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / max(args.steps, 1), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": {akmc.PREC_FP32: "fp32-equivalent (3x fp16 tcgen05, fp32 accumulate) + fp64 selection",
                          akmc.PREC_FP16_FAST: "fp16 single pass (tcgen05, fp32 accumulate; information only, "
                                               "fails the 1e-5 rate bar) + fp64 selection"}.get(prec, "f64"),
                "data": "synthetic",
                "config": {"workload": args.workload.upper(), "cells_per_gpu": list(cfg.cells),
                           "voxels_per_gpu": cfg.n_voxels, "sites_per_gpu": sites,
                           "vacancies_per_gpu": pr.n_vac_per_voxel * cfg.n_voxels,
                           "domain_cells": list(cfg.domain_cells), "lambda": args.lam, "window_s": cfg.window_s,
                           "step": ("one sweep (8 sublattice phases)" if pr.domain[0] else
                                    f"{nstep} world-model events per voxel (one world-kernel launch)" if wnets else
                                    f"{nstep} BKL events per voxel (one engine launch)"),
                           "temperature_K": ("per voxel, uniform 558-577" if vT is not None else cfg.temperature_K),
                           "model": ("world-model mode: policy logits -E/kT of the physics-embedded MLP (tau_act 1), "
                                     f"Eq. 7 clock from a seeded Poisson-time net (H = {WORLD_H}), FP64" if wnets else
                                     "MLP 448-256-256-8 physics-embedded + residual" if model else "pair KRA"),
                           "parallelism": ("1 GPU" if world == 1 else
                                           (f"spatial blocks {'x'.join(map(str, cfg.gpu_grid))}, halo deltas between "
                                            "phases written into the peers' mailboxes over NVLink (CUDA IPC)" if cfg.world > 1 else f"independent voxels x{world}")),
                           "l2": "inputs > L2 (lattice %.2f GB per GPU)" % (sites / 1e9)},
                "sim_seconds_per_wall_second": (sim_s * world / world) / (ms_max / 1e3),
                "events_per_s": float(sm[2]) / (ms_max / 1e3),
                "executed_hop_evals_per_s": (8.0 * mlp_rows / (prof_ms / 1e3)) if prof_ms > 0 else None,
                "executed_note": "hop evaluations whose network row actually ran (memo misses; instrumented pass) per "
                                 "second -- `value` counts the method's logical evaluations (R4), of which the exact "
                                 "per-vacancy memo (R7) serves the rest",
                "gpu_launches": int(float(sm[6])),
                "roofline": roof,
                "e2e": {"value": e2e_value, "unit": UNIT,
                        "h2d_bytes_per_step": int(sites / max(args.steps, 1)),
                        "d2h_bytes_per_step": int(sites / max(args.steps, 1)) + 88,
                        "parts": e2e_parts,
                "note": "akmc_init from pinned host lattice + K x (akmc_step + counters readback) + "
                                "final akmc_state lattice readback (canonical order), host wall clock"},
                "clocks": cs.summary()}
    if world > 1:
        dist.barrier()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb, _, _ = cpu_baseline(args.workload, 1, args.lam, world=bool(wnets))
        if not wnets:
            cb["all_cores"] = cpu_baseline_all_cores(args.workload, args.lam)
        line["cpu_baseline"] = cb
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    os.environ.pop("NCCL_DEBUG", None)              # keep NCCL's version banner off stdout (one JSON line)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64", "fast"],
                    help="fast = single-pass fp16 layers 2-3 (information only: fails the 1e-5 rate bar)")
    ap.add_argument("--model", default="mlp", choices=["mlp", "pair"])
    ap.add_argument("--lam", type=float, default=0.25)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--events", type=int, default=100, help="serial workloads: BKL events per voxel per step")
    ap.add_argument("--voxel-T", action="store_true", help="per-voxel temperature uniform in 558-577 K (C4 variant)")
    ap.add_argument("--replicas", type=int, default=0,
                    help="serial workloads: this many independent replica voxels per GPU (e.g. C1 x 4096)")
    ap.add_argument("--world", action="store_true",
                    help="serial workloads: the world-model time mode (SURVEY 8(f) f2; FP64: policy logits -E/kT of the "
                         "physics network, Eq. 7 clock from a seeded Poisson-time net)")
    ap.add_argument("--ramp-s", type=float, default=1.0, help="untimed clock ramp before the warm-up steps")
    args = ap.parse_args()
    global REPLICAS
    REPLICAS = args.replicas or None
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
