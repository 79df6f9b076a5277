"""Parity at BASELINE.json's full size (C5: 1024^3 cells, 214,748 vacancies, FP32-equivalent MLP, domains 8^3,
lambda = 1/4) in the launch configuration bench.py times, via sampled outputs the oracle computes one by one
and properties that hold at any size:
  * species counts are conserved and the vacancy registry equals the set of V sites;
  * every voxel clock advanced by exactly 2 windows (2 sweeps; A19/A25);
  * the rates of sampled vacancies (after the sweeps) equal the FP64 oracle's within 1e-5 relative.
Plus the FP64 pair-model trajectories at the full C3 (512^3, 26,844 vacancies, 2 sweeps) and C5 (1024^3, 214,748
vacancies, 1 sweep) sizes, bit-exact against the oracle: the engine's refill from millions of domains, the fair-
share claims and the hot/cold segment lists run here exactly as in the bench.
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

RTOL_FAST = 1e-5


@pytest.fixture(scope="module")
def akmc():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_24091_b200 as A
    from paper_2604_24091_b200 import build
    build.build()
    return A


def test_c5_fullsize_sweeps(akmc, orc):
    import torch
    import bench
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=1)
    cfg, pr = bench.sim_config("c5", akmc.PREC_FP32, akmc.MODEL_MLP, 0.25, E0)
    sp, keep = bench.make_inputs("c5", 0, torch.device("cuda", 0))
    counts0 = np.bincount(sp, minlength=7)
    assert counts0[6] == pr.n_vac_per_voxel
    with akmc.Simulation(cfg, sp, eps, E0, mlp) as sim:
        c = sim.step(2)
        gsp, gvac, gclock, gctr = sim.state()
        G, E = sim.rates()
    assert c["events"] > 100000
    assert np.array_equal(np.bincount(gsp, minlength=7), counts0)
    assert np.array_equal(np.sort(gvac), np.flatnonzero(gsp == 6))
    assert gclock[0] == 2 * cfg.window_s
    ocfg = orc.Config(cells=cfg.cells, n_voxels=1, T=cfg.temperature_K, nu0=cfg.nu0, kB=cfg.kB, model=1,
                      domain=cfg.domain_cells, window_s=cfg.window_s, seed=cfg.seed)
    rng = np.random.default_rng(7)
    idx = rng.choice(gvac.size, size=256, replace=False)
    worst = 0.0
    for i in idx:
        _, g_orc, _ = orc.barriers(ocfg, gsp, int(gvac[i]), mlp=mlp)
        scale = np.maximum(np.abs(g_orc), 1e-300)
        rel = np.where(g_orc == 0.0, np.abs(G[i]), np.abs(G[i] - g_orc) / scale)
        worst = max(worst, float(rel.max()))
        assert np.array_equal(G[i] == 0.0, g_orc == 0.0)          # masks exact
    assert worst <= RTOL_FAST, worst


@pytest.mark.parametrize("name,sweeps,dataflow", [("c3", 2, False), ("c5", 1, False), ("c5", 1, True)])
def test_fullsize_fp64_pair_bitexact(akmc, orc, name, sweeps, dataflow):
    import torch
    import bench
    eps, E0 = synth.illustrative_pair_params()
    cfg, pr = bench.sim_config(name, akmc.PREC_FP64, akmc.MODEL_PAIR, 0.25, E0)
    sp, keep = bench.make_inputs(name, 0, torch.device("cuda", 0))
    sp = np.ascontiguousarray(sp)
    with akmc.Simulation(cfg, sp, eps, E0) as sim:
        if dataflow:
            sim.set_dataflow(True)                   # f1: tile readiness instead of phase boundaries
        c = sim.step(sweeps)
        gsp, gvac, gclock, gctr = sim.state()
    del keep
    ocfg = orc.Config(cells=cfg.cells, n_voxels=1, T=cfg.temperature_K, nu0=cfg.nu0, kB=cfg.kB, model=0,
                      domain=cfg.domain_cells, window_s=cfg.window_s, seed=cfg.seed)
    st = orc.State.from_species(ocfg, sp)
    del sp
    orc.run(ocfg, st, sweeps, eps, E0)
    assert c["events"] > 10000
    assert gctr["events"] == st.counters[0] and gctr["hop_evals"] == st.counters[1]
    assert np.array_equal(gvac, st.vac)
    assert np.array_equal(gclock, st.clock)
    assert np.array_equal(gsp, st.species)
