"""GPU parity tests: the CUDA path (through the C-ABI) against the FP64 CPU oracle.

Bars (north star): integer lattice trajectories bit-exact in FP64 mode with the same Philox
stream; per-hop rates of the tensor-core FP32-equivalent mode within 1e-5 relative.
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

RTOL_FAST = 1e-5        # north star: reduced-precision per-hop rates within 1e-5 relative


@pytest.fixture(scope="module")
def akmc():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_24091_b200 as A
    from paper_2604_24091_b200 import build
    build.build()
    return A


def _params():
    eps, E0 = synth.illustrative_pair_params()
    return eps, E0


def _ocfg(orc, acfg):
    return orc.Config(cells=acfg.cells, n_voxels=acfg.n_voxels, T=acfg.temperature_K, nu0=acfg.nu0, kB=acfg.kB,
                      model=acfg.barrier_model, domain=acfg.domain_cells, window_s=acfg.window_s, seed=acfg.seed)


# ----------------------------------------------------------------------------- deterministic exp / log
def test_det_exp_log_bitexact_vs_oracle(akmc, orc):
    """the device det_exp / det_log (A29) equal the oracle's bit for bit on 2e7 arguments
    spanning the ranges the path uses (-E/kT in [-60, 0] plus the tail to -700; u = k 2^-53 in (0, 1])."""
    rng = np.random.default_rng(2604)
    n = 10_000_000
    xe = np.concatenate([-rng.random(n) * 60.0, -rng.random(n // 10) * 700.0, [0.0, -0.0, -1e-300, -5e-324]])
    ye = akmc.debug_math(0, xe)
    assert np.array_equal(ye.view(np.uint64), orc.det_exp_n(xe).view(np.uint64))
    # Philox uniforms are multiples of 2^-53 in (0, 1]
    u = np.concatenate([(rng.integers(0, 2 ** 53, n, dtype=np.int64) + 1).astype(np.float64) * 2.0 ** -53,
                        2.0 ** -rng.integers(0, 54, n // 10).astype(np.float64), [1.0, 2.0 ** -53]])
    yl = akmc.debug_math(1, u)
    assert np.array_equal(yl.view(np.uint64), orc.det_log_n(u).view(np.uint64))


# ----------------------------------------------------------------------------- network evaluation
@pytest.mark.parametrize("weights", ["random", "physics_residual"])
def test_eval_windows_fp64_bitexact(akmc, orc, weights):
    eps, E0 = _params()
    mlp = synth.random_mlp(seed=3) if weights == "random" else synth.physics_mlp(eps, E0, residual=0.02, seed=4)
    wins = synth.random_windows(1000, seed=5)
    cfg = akmc.Config(cells=(8, 8, 8), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP64)
    with akmc.Simulation(cfg, np.zeros(1024, np.uint8), mlp=mlp) as sim:
        E = sim.eval_windows(wins, akmc.PREC_FP64)
    ref = np.stack([orc.mlp_fp64(w, mlp) for w in wins])
    assert np.array_equal(E, ref)


@pytest.mark.parametrize("weights", ["random", "physics", "physics_residual"])
@pytest.mark.parametrize("n", [1, 127, 128, 4096 + 77])
def test_eval_windows_fp32_tensor_core(akmc, orc, weights, n):
    """tcgen05 FP32-equivalent barrier network: rates within 1e-5 relative of FP64 (every hop),
    tiles of 128 plus a ragged tail."""
    eps, E0 = _params()
    mlp = {"random": lambda: synth.random_mlp(seed=7),
           "physics": lambda: synth.physics_mlp(eps, E0),
           "physics_residual": lambda: synth.physics_mlp(eps, E0, residual=0.02, seed=8)}[weights]()
    wins = synth.random_windows(n, seed=9 + n)
    cfg = akmc.Config(cells=(8, 8, 8), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32)
    with akmc.Simulation(cfg, np.zeros(1024, np.uint8), mlp=mlp) as sim:
        E32 = sim.eval_windows(wins, akmc.PREC_FP32)
    ref = np.stack([orc.mlp_fp64(w, mlp) for w in wins])
    kT = cfg.kB * cfg.temperature_K
    rel = np.abs(np.expm1(-(E32 - ref) / kT))
    assert rel.max() <= RTOL_FAST, (rel.max(), np.abs(E32 - ref).max())


# ----------------------------------------------------------------------------- rates on lattices
@pytest.mark.parametrize("model", ["pair", "mlp"])
def test_rates_fp64_bitexact(akmc, orc, model):
    eps, E0 = _params()
    L = 16
    sp = synth.make_lattice((L, L, L), 2, synth.a508_atomic_fractions(), 12, seed=11)
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=1) if model == "mlp" else None
    cfg = akmc.Config(cells=(L, L, L), n_voxels=2, barrier_model=akmc.MODEL_PAIR if model == "pair" else akmc.MODEL_MLP,
                      precision=akmc.PREC_FP64)
    with akmc.Simulation(cfg, sp, eps, E0, mlp) as sim:
        R, E = sim.rates()
        _, vac, _, _ = sim.state(species=False)
    oc = _ocfg(orc, cfg)
    Ro, Eo = orc.rates(oc, sp, vac, eps, E0, mlp)
    assert np.array_equal(R, Ro)
    assert np.array_equal(E, Eo)


def test_rates_fp32_lattice(akmc, orc):
    eps, E0 = _params()
    L = 24
    sp = synth.make_lattice((L, L, L), 1, synth.a508_atomic_fractions(), 200, seed=12)
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=2)
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32)
    with akmc.Simulation(cfg, sp, mlp=mlp) as sim:
        R, E = sim.rates()
        _, vac, _, _ = sim.state(species=False)
    Ro, Eo = orc.rates(_ocfg(orc, cfg), sp, vac, None, None, mlp)
    assert np.array_equal(R == 0, Ro == 0)           # masks identical
    m = Ro > 0
    assert np.max(np.abs(R[m] / Ro[m] - 1)) <= RTOL_FAST


def test_fp16_fast_mode_information_only(akmc, orc):
    """SURVEY 8(b) fast mode (single fp16 pass on layers 2-3): rates within 3e-2 relative of the FP64 oracle on
    30 %-solute windows (measured max ~1.0e-2; it is NOT held to the 1e-5 bar), the FP32-equivalent mode is
    strictly more accurate on the same windows,
    masks identical; a sublattice run in fast mode conserves species and keeps the registry consistent."""
    eps, E0 = _params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=8)
    wins = synth.random_windows(3000, seed=12)
    cfg = akmc.Config(cells=(8, 8, 8), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP16_FAST)
    with akmc.Simulation(cfg, np.zeros(1024, np.uint8), mlp=mlp) as sim:
        Ef = sim.eval_windows(wins, akmc.PREC_FP16_FAST)
        E32 = sim.eval_windows(wins, akmc.PREC_FP32)
    ref = np.stack([orc.mlp_fp64(w, mlp) for w in wins])
    kT = cfg.kB * cfg.temperature_K
    rel_f = np.abs(np.expm1(-(Ef - ref) / kT))
    rel_32 = np.abs(np.expm1(-(E32 - ref) / kT))
    assert rel_f.max() <= 3e-2, rel_f.max()
    assert rel_32.max() <= RTOL_FAST and rel_32.max() < rel_f.max()
    L = 24
    sp = synth.make_lattice((L, L, L), 1, synth.a508_atomic_fractions(), 60, seed=13)
    cfg2 = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP16_FAST,
                       domain_cells=(8, 8, 8), window_s=synth.window_seconds(1.0, E0[0]), seed=3)
    with akmc.Simulation(cfg2, sp, mlp=mlp) as sim:
        c = sim.step(4)
        gsp, gvac, _, _ = sim.state()
        R, _ = sim.rates()
    assert c["events"] > 20
    assert np.array_equal(np.bincount(gsp, minlength=7), np.bincount(sp, minlength=7))
    assert np.array_equal(np.sort(np.flatnonzero(gsp == 6)), np.sort(gvac))
    assert np.all(R >= 0)


# ----------------------------------------------------------------------------- trajectories
def _run_both(akmc, orc, cfg, sp, n, eps=None, E0=None, mlp=None, chunks=1):
    ost = orc.State.from_species(_ocfg(orc, cfg), sp)
    with akmc.Simulation(cfg, sp, eps, E0, mlp) as sim:
        for _ in range(chunks):
            c = sim.step(n // chunks)
            orc.run(_ocfg(orc, cfg), ost, n // chunks, eps, E0, mlp)
        gsp, gvac, gclock, gctr = sim.state()
    return ost, (gsp, gvac, gclock, gctr)


def test_serial_C1_bitexact_1e4_steps(akmc, orc):
    """C1: Fe-1at%Cu 16^3, 1 vacancy, 10^4 BKL steps at 563 K, pair model FP64: bit-exact."""
    eps, E0 = _params()
    pr = synth.preset("C1")
    sp = synth.make_lattice(pr.cells, 1, pr.fractions, 1, seed=pr.seed)
    cfg = akmc.Config(cells=pr.cells, barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=2605)
    ost, (gsp, gvac, gclock, gctr) = _run_both(akmc, orc, cfg, sp, 10000, eps, E0, chunks=4)
    assert np.array_equal(gsp, ost.species)
    assert np.array_equal(gvac, ost.vac)
    assert np.array_equal(gclock, ost.clock)
    assert gctr["events"] == ost.counters[0] == 10000
    assert gctr["hop_evals"] == ost.counters[1]


def test_serial_mlp_fp64_bitexact(akmc, orc):
    eps, E0 = _params()
    L = 16
    sp = synth.make_lattice((L, L, L), 1, synth.fe_cu_fractions(0.03), 3, seed=21)
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=3)
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP64, seed=77)
    ost, (gsp, gvac, gclock, gctr) = _run_both(akmc, orc, cfg, sp, 600, mlp=mlp)
    assert np.array_equal(gsp, ost.species)
    assert np.array_equal(gvac, ost.vac)
    assert np.array_equal(gclock, ost.clock)


def test_voxel_batch_bitexact(akmc, orc):
    """C4-shaped (reduced): independent periodic voxels, one BKL competing set each."""
    eps, E0 = _params()
    L = 16
    nvox = 12
    sp = synth.make_lattice((L, L, L), nvox, synth.a508_atomic_fractions(), 10, seed=31)
    cfg = akmc.Config(cells=(L, L, L), n_voxels=nvox, barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=5)
    ost, (gsp, gvac, gclock, gctr) = _run_both(akmc, orc, cfg, sp, 300, eps, E0)
    assert np.array_equal(gsp, ost.species)
    assert np.array_equal(gvac, ost.vac)
    assert np.array_equal(gclock, ost.clock)
    assert gctr["events"] == ost.counters[0]


@pytest.mark.parametrize("model", ["pair", "mlp"])
def test_anisotropic_cells_serial_bitexact(akmc, orc, model):
    """Geometry edge case: Lx != Ly != Lz and none a multiple of the 4-cell brick (S:30 asks only even,
    >= 4), so the last brick along every axis is ragged and a transposed axis or stride in the periodic
    wrap / brick index would move a hop to the wrong site.  Three voxels, FP64, bit-exact vs the oracle."""
    eps, E0 = _params()
    cells, nvox = (6, 10, 14), 3
    sp = synth.make_lattice(cells, nvox, synth.a508_atomic_fractions(), 4, seed=71)
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=7) if model == "mlp" else None
    cfg = akmc.Config(cells=cells, n_voxels=nvox, barrier_model=akmc.MODEL_PAIR if model == "pair" else akmc.MODEL_MLP,
                      precision=akmc.PREC_FP64, seed=23)
    if mlp is None:
        ost, (gsp, gvac, gclock, gctr) = _run_both(akmc, orc, cfg, sp, 400, eps, E0, chunks=2)
    else:
        ost, (gsp, gvac, gclock, gctr) = _run_both(akmc, orc, cfg, sp, 200, mlp=mlp, chunks=2)
    assert np.array_equal(gsp, ost.species)
    assert np.array_equal(gvac, ost.vac)
    assert np.array_equal(gclock, ost.clock)
    assert gctr["events"] == ost.counters[0]


def test_anisotropic_domains_sublattice_bitexact(akmc, orc):
    """Sublattice mode on a non-cubic lattice with non-cubic domains (18 x 24 x 30 cells, 6 x 8 x 10-cell
    domains, so 3 x 3 x 3 domains with sectors of 3 x 4 x 5 cells, A20) and ragged bricks along x and z:
    the sector permutation, activation and window bookkeeping per axis.  FP64 pair, 6 sweeps, bit-exact."""
    eps, E0 = _params()
    cells = (18, 24, 30)
    sp = synth.make_lattice(cells, 1, synth.a508_atomic_fractions(), 60, seed=73)
    cfg = akmc.Config(cells=cells, barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=29,
                      domain_cells=(6, 8, 10), window_s=synth.window_seconds(1.0, E0[0]))
    ost, (gsp, gvac, gclock, gctr) = _run_both(akmc, orc, cfg, sp, 6, eps, E0, chunks=2)
    assert np.array_equal(gsp, ost.species)
    assert np.array_equal(gvac, ost.vac)
    assert np.array_equal(gclock, ost.clock)
    assert gctr["events"] == ost.counters[0] and gctr["hop_evals"] == ost.counters[1]
    assert ost.counters[0] > 0


@pytest.mark.parametrize("mode", ["serial", "voxels", "sublattice"])
def test_zero_rate_vacancy_bitexact(akmc, orc, mode):
    """Degenerate input: a vacancy whose eight first neighbours are vacancies (every hop masked, R_i = 0,
    A14) inside the competing set -- the zero leaf of the pairwise tree and the descent guards (A17).
    FP64 pair trajectories bit-exact vs the oracle in serial, voxel-batch and sublattice mode; FP32
    tensor-core rates have the oracle's masks (the centre's row all zero) and stay within 1e-5."""
    eps, E0 = _params()
    L = 16
    nvox = 4 if mode == "voxels" else 1
    base = synth.make_lattice((L, L, L), nvox, synth.fe_cu_fractions(0.05), 3, seed=61)
    S = 2 * L ** 3
    sp = base.copy()
    for v in range(nvox):
        sp[v * S:(v + 1) * S], _ = synth.with_vacancy_cluster(base[v * S:(v + 1) * S], (L, L, L), (5 + v, 6, 7))
    dom, win = ((8, 8, 8), synth.window_seconds(1.0, E0[0])) if mode == "sublattice" else ((0, 0, 0), 0.0)
    cfg = akmc.Config(cells=(L, L, L), n_voxels=nvox, barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64,
                      seed=17, domain_cells=dom, window_s=win)
    n = 10 if mode == "sublattice" else 400
    ost, (gsp, gvac, gclock, gctr) = _run_both(akmc, orc, cfg, sp, n, eps, E0, chunks=2)
    assert ost.counters[0] > 20
    assert np.array_equal(gsp, ost.species)
    assert np.array_equal(gvac, ost.vac)
    assert np.array_equal(gclock, ost.clock)
    assert gctr["events"] == ost.counters[0]
    assert gctr["hop_evals"] == ost.counters[1]
    if mode != "serial":
        return
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=9)
    cfg32 = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32)
    with akmc.Simulation(cfg32, sp, mlp=mlp) as sim:
        R, _ = sim.rates()
        _, vac, _, _ = sim.state(species=False)
    Ro, _ = orc.rates(_ocfg(orc, cfg32), sp, vac, None, None, mlp)
    assert np.array_equal(R == 0, Ro == 0)
    assert np.any(np.all(Ro == 0, axis=1))           # the centre row is fully masked
    m = Ro > 0
    assert np.max(np.abs(R[m] / Ro[m] - 1)) <= RTOL_FAST


def test_voxel_batch_empty_voxel(akmc, orc):
    """Ragged voxel batch: the middle voxel holds no vacancy (empty competing set) while its
    neighbours in the batch keep stepping.  The call reports AKMC_TERMINAL like the oracle, the empty voxel's
    clock stays 0, and the other voxels' trajectories are bit-exact."""
    eps, E0 = _params()
    L, nvox = 8, 3
    S = 2 * L ** 3
    sp = synth.make_lattice((L, L, L), nvox, synth.fe_cu_fractions(0.05), 3, seed=5)
    mid = sp[S:2 * S]
    mid[mid == 6] = 0
    cfg = akmc.Config(cells=(L, L, L), n_voxels=nvox, barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=4)
    ost = orc.State.from_species(_ocfg(orc, cfg), sp)
    orc_rc = orc.run(_ocfg(orc, cfg), ost, 50, eps, E0)
    with akmc.Simulation(cfg, sp, eps, E0) as sim:
        c = sim.step(50)
        gsp, gvac, gclock, gctr = sim.state()
    assert orc_rc == akmc.AKMC_TERMINAL and c["status"] == akmc.AKMC_TERMINAL
    assert ost.counters[0] == 100 and gctr["events"] == 100
    assert gclock[1] == 0.0
    assert np.array_equal(gsp, ost.species)
    assert np.array_equal(gvac, ost.vac)
    assert np.array_equal(gclock, ost.clock)


@pytest.mark.parametrize("model", ["pair", "mlp"])
def test_voxel_batch_heterogeneous_T_bitexact(akmc, orc, model):
    """C4 variant: per-voxel T uniform in 558-577 K; FP64 trajectories bit-exact vs the
    oracle with the same per-voxel T, including a temperature change between steps (memo cleared)."""
    eps, E0 = _params()
    L = 16
    nvox = 10
    sp = synth.make_lattice((L, L, L), nvox, synth.a508_atomic_fractions(), 10, seed=33)
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=4) if model == "mlp" else None
    T1 = synth.voxel_temperatures(nvox, seed=2608)
    T2 = synth.voxel_temperatures(nvox, seed=2609)
    cfg = akmc.Config(cells=(L, L, L), n_voxels=nvox, precision=akmc.PREC_FP64, seed=6,
                      barrier_model=akmc.MODEL_PAIR if model == "pair" else akmc.MODEL_MLP)
    n = 200 if model == "pair" else 40
    oc1 = orc.Config(**{**_ocfg(orc, cfg).__dict__, "voxel_T": T1})
    oc2 = orc.Config(**{**_ocfg(orc, cfg).__dict__, "voxel_T": T2})
    ost = orc.State.from_species(oc1, sp)
    with akmc.Simulation(cfg, sp, eps, E0, mlp) as sim:
        sim.set_voxel_temperatures(T1)
        sim.step(n)
        R, _ = sim.rates()
        orc.run(oc1, ost, n, eps, E0, mlp)
        Ro, _ = orc.rates(oc1, ost.species, ost.vac, eps, E0, mlp)
        assert np.array_equal(R, Ro)
        sim.set_voxel_temperatures(T2)
        sim.step(n)
        orc.run(oc2, ost, n, eps, E0, mlp)
        gsp, gvac, gclock, gctr = sim.state()
        with pytest.raises(akmc.AkmcError):
            sim.set_voxel_temperatures(T2[:-1])
    assert np.array_equal(gsp, ost.species)
    assert np.array_equal(gvac, ost.vac)
    assert np.array_equal(gclock, ost.clock)
    assert gctr["events"] == ost.counters[0]


@pytest.mark.parametrize("model", ["pair", "mlp"])
def test_run_until_voxel_ensemble_bitexact(akmc, orc, model):
    """Voxel-ensemble mode with per-voxel T: every voxel advanced to a common physical time in
    two horizons (and an event cap) -- bit-exact vs the oracle's run_until."""
    eps, E0 = _params()
    L = 16
    nvox = 12
    sp = synth.make_lattice((L, L, L), nvox, synth.a508_atomic_fractions(), 10, seed=35)
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=6) if model == "mlp" else None
    T = synth.voxel_temperatures(nvox, seed=2611)
    cfg = akmc.Config(cells=(L, L, L), n_voxels=nvox, precision=akmc.PREC_FP64, seed=8,
                      barrier_model=akmc.MODEL_PAIR if model == "pair" else akmc.MODEL_MLP)
    oc = orc.Config(**{**_ocfg(orc, cfg).__dict__, "voxel_T": T})
    t1, t2 = 5e-9, 1.5e-8                            # ~ 6 / 20 events per voxel
    ost = orc.State.from_species(oc, sp)
    with akmc.Simulation(cfg, sp, eps, E0, mlp) as sim:
        sim.set_voxel_temperatures(T)
        sim.run_until(t1)
        orc.run_until(oc, ost, t1, 10 ** 9, eps, E0, mlp)
        _, _, gclock1, _ = sim.state(species=False)
        assert np.array_equal(gclock1, ost.clock) and np.all(gclock1 <= t1)
        sim.run_until(t2, max_events=7)              # the cap binds for the busiest voxels
        orc.run_until(oc, ost, t2, 7, eps, E0, mlp)
        sim.run_until(t2)
        orc.run_until(oc, ost, t2, 10 ** 9, eps, E0, mlp)
        gsp, gvac, gclock, gctr = sim.state()
    assert np.array_equal(gsp, ost.species)
    assert np.array_equal(gvac, ost.vac)
    assert np.array_equal(gclock, ost.clock)
    assert np.all(gclock <= t2)
    assert gctr["events"] == ost.counters[0] > 10 * nvox
    assert gctr["hop_evals"] == ost.counters[1]


def test_rates_fp32_heterogeneous_T(akmc, orc):
    """Tensor-core FP32 rates at per-voxel T within 1e-5 of the FP64 oracle at the same T."""
    eps, E0 = _params()
    L = 16
    nvox = 6
    sp = synth.make_lattice((L, L, L), nvox, synth.a508_atomic_fractions(), 40, seed=34)
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=5)
    T = synth.voxel_temperatures(nvox, seed=2610)
    cfg = akmc.Config(cells=(L, L, L), n_voxels=nvox, barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32)
    with akmc.Simulation(cfg, sp, mlp=mlp) as sim:
        sim.set_voxel_temperatures(T)
        R, _ = sim.rates()
        _, vac, _, _ = sim.state(species=False)
    Ro, _ = orc.rates(orc.Config(**{**_ocfg(orc, cfg).__dict__, "voxel_T": T}), sp, vac, None, None, mlp)
    assert np.array_equal(R == 0, Ro == 0)
    m = Ro > 0
    assert np.max(np.abs(R[m] / Ro[m] - 1)) <= RTOL_FAST


@pytest.mark.parametrize("lam,driver", [(1.0, "graph"), (0.25, "graph"), (1.0, "host")])
def test_sublattice_bitexact(akmc, orc, lam, driver):
    """Windowed synchronous sublattice (reading A19), domains 8^3: bit-exact vs the oracle, with the
    per-sweep CUDA graph (device-side inner loop) and with the host-stepped (profiling) driver."""
    eps, E0 = _params()
    L = 32
    sp = synth.make_lattice((L, L, L), 1, synth.fe_cu_fractions(0.05), 60, seed=41)
    win = synth.window_seconds(lam, E0[0])
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=9,
                      domain_cells=(8, 8, 8), window_s=win)
    ost = orc.State.from_species(_ocfg(orc, cfg), sp)
    with akmc.Simulation(cfg, sp, eps, E0) as sim:
        sim.set_profiling(driver == "host")
        for _ in range(2):
            sim.step(4)
            orc.run(_ocfg(orc, cfg), ost, 4, eps, E0)
        gsp, gvac, gclock, gctr = sim.state()
    assert ost.counters[0] > 20
    assert np.array_equal(gsp, ost.species)
    assert np.array_equal(gvac, ost.vac)
    assert np.array_equal(gclock, ost.clock)
    assert gctr["events"] == ost.counters[0]
    assert gctr["hop_evals"] == ost.counters[1]


def test_sublattice_bitexact_1e4_events(akmc, orc):
    """North-star bar in sublattice mode: >= 10^4 events (200 sweeps, 300 vacancies in the A508 alloy, 8^3
    domains, lambda = 1) bit-exact vs the oracle -- lattice, vacancy registry, clock and counters -- with the
    state compared after every 40 sweeps."""
    eps, E0 = _params()
    L = 32
    sp = synth.make_lattice((L, L, L), 1, synth.a508_atomic_fractions(), 300, seed=91)
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=12,
                      domain_cells=(8, 8, 8), window_s=synth.window_seconds(1.0, E0[0]))
    ost = orc.State.from_species(_ocfg(orc, cfg), sp)
    with akmc.Simulation(cfg, sp, eps, E0) as sim:
        for _ in range(5):
            sim.step(40)
            orc.run(_ocfg(orc, cfg), ost, 40, eps, E0)
            gsp, gvac, gclock, gctr = sim.state()
            assert np.array_equal(gsp, ost.species)
            assert np.array_equal(gvac, ost.vac)
            assert np.array_equal(gclock, ost.clock)
            assert gctr["events"] == ost.counters[0] and gctr["hop_evals"] == ost.counters[1]
    assert ost.counters[0] >= 10_000


def test_sublattice_mlp_fp64_bitexact(akmc, orc):
    eps, E0 = _params()
    L = 24
    sp = synth.make_lattice((L, L, L), 1, synth.a508_atomic_fractions(), 40, seed=42)
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=6)
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP64, seed=19,
                      domain_cells=(6, 6, 6), window_s=synth.window_seconds(1.0, E0[0]))
    ost, (gsp, gvac, gclock, gctr) = _run_both(akmc, orc, cfg, sp, 3, mlp=mlp)
    assert np.array_equal(gsp, ost.species)
    assert np.array_equal(gvac, ost.vac)


def test_terminal_and_conservation(akmc):
    L = 8
    sp = np.zeros(2 * L ** 3, np.uint8)
    eps, E0 = _params()
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_PAIR)
    with akmc.Simulation(cfg, sp, eps, E0) as sim:
        c = sim.step(5)
        assert c["status"] == akmc.AKMC_TERMINAL
        gsp, vac, clock, _ = sim.state()
        assert np.array_equal(gsp, sp) and clock[0] == 0.0


def test_sublattice_no_vacancy(akmc, orc):
    """Empty input in sublattice mode: no vacancy in any domain.  Every phase is empty, each sweep still
    advances the global clock by the window (A19/A22), no event, lattice unchanged -- as the oracle does."""
    eps, E0 = _params()
    L = 16
    sp = np.zeros(2 * L ** 3, np.uint8)
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=3,
                      domain_cells=(8, 8, 8), window_s=synth.window_seconds(1.0, E0[0]))
    ost = orc.State.from_species(_ocfg(orc, cfg), sp)
    orc_rc = orc.run(_ocfg(orc, cfg), ost, 3, eps, E0)
    with akmc.Simulation(cfg, sp, eps, E0) as sim:
        c = sim.step(3)
        gsp, gvac, gclock, gctr = sim.state()
    assert orc_rc == 0 and c["status"] == akmc.AKMC_OK
    assert np.array_equal(gsp, sp) and gvac.size == 0
    assert np.array_equal(gclock, ost.clock) and gctr["events"] == 0
    # the tensor-core evaluator path with zero rows: FP32 MLP sublattice step and akmc_rates
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=9)
    cfg32 = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32, seed=3,
                        domain_cells=(8, 8, 8), window_s=synth.window_seconds(1.0, E0[0]))
    with akmc.Simulation(cfg32, sp, mlp=mlp) as sim:
        c = sim.step(2)
        R, E = sim.rates()
        gsp, gvac, gclock, gctr = sim.state()
    assert c["status"] == akmc.AKMC_OK and R.shape == (0, 8) and E.shape == (0, 8)
    assert np.array_equal(gsp, sp) and gvac.size == 0 and gctr["events"] == 0
    assert gclock[0] == 2 * cfg32.window_s


@pytest.mark.parametrize("mode", ["serial", "sublattice"])
def test_vacancy_cap_bitexact(akmc, orc, mode):
    """Maximum size of the vacancy list: exactly 1 % of the sites (one more is AKMC_ERR_INVALID).
    16^3 cells, 81 vacancies: ~10 per 8^3 domain (multi-slot competing sets) in sublattice mode, one
    81-member competing set in serial mode.  FP64 pair trajectories bit-exact vs the oracle."""
    eps, E0 = _params()
    L = 16
    nv = int(0.01 * 2 * L ** 3)
    sp = synth.make_lattice((L, L, L), 1, synth.a508_atomic_fractions(), nv, seed=73)
    dom, win = ((8, 8, 8), synth.window_seconds(0.25, E0[0])) if mode == "sublattice" else ((0, 0, 0), 0.0)
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=29,
                      domain_cells=dom, window_s=win)
    n = 6 if mode == "sublattice" else 500
    ost, (gsp, gvac, gclock, gctr) = _run_both(akmc, orc, cfg, sp, n, eps, E0, chunks=2)
    assert gvac.size == nv and ost.counters[0] > 50
    assert np.array_equal(gsp, ost.species)
    assert np.array_equal(gvac, ost.vac)
    assert np.array_equal(gclock, ost.clock)
    assert gctr["events"] == ost.counters[0]
    assert gctr["hop_evals"] == ost.counters[1]
    sp2 = sp.copy()
    sp2[np.flatnonzero(sp2 != 6)[0]] = 6
    with pytest.raises(akmc.AkmcError):
        akmc.Simulation(cfg, sp2, eps, E0)


# ----------------------------------------------------------------------------- phase engine specifics
def _crowded_lattice(L, n_spread, cluster_center, n_cluster, seed):
    """Fe-5%Cu lattice with n_spread random vacancies plus n_cluster vacancies packed around one site, so
    that some domains hold > 2 vacancies (multi-slot placement) and one holds > 16 (tree in scratch)."""
    sp = synth.make_lattice((L, L, L), 1, synth.fe_cu_fractions(0.05), n_spread, seed=seed)
    rng = np.random.default_rng(seed + 1)
    cx, cy, cz = cluster_center
    placed = 0
    while placed < n_cluster:
        x, y, z = (int(v) for v in rng.integers(-2, 3, size=3))
        b = int(rng.integers(0, 2))
        i = 2 * (((cx + x) % L) + L * (((cy + y) % L) + L * ((cz + z) % L))) + b
        if sp[i] != 6:
            sp[i] = 6
            placed += 1
    return sp


@pytest.mark.parametrize("lam", [1.0, 0.25])
def test_engine_crowded_domains_bitexact(akmc, orc, lam):
    """Domains with many vacancies: multi-slot placement, carried-over (pending) domains and > 16-member
    competing sets (tree in global scratch) stay bit-exact vs the oracle."""
    eps, E0 = _params()
    L = 32
    sp = _crowded_lattice(L, 120, (12, 12, 12), 40, seed=77)
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=23,
                      domain_cells=(8, 8, 8), window_s=synth.window_seconds(lam, E0[0]))
    ost, (gsp, gvac, gclock, gctr) = _run_both(akmc, orc, cfg, sp, 4, eps=eps, E0=E0)
    assert ost.counters[0] > 50
    assert np.array_equal(gsp, ost.species)
    assert np.array_equal(gvac, ost.vac)
    assert np.array_equal(gclock, ost.clock)
    assert gctr["events"] == ost.counters[0] and gctr["hop_evals"] == ost.counters[1]


def test_engine_evaluator_row_purity(akmc):
    """The FP32-equivalent evaluator's result for a window does not depend on the tile it is evaluated in
    (order, neighbours, batch size): the property that makes the per-vacancy memo and any decomposition
    exact."""
    eps, E0 = _params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=4)
    rng = np.random.default_rng(5)
    w = synth.random_windows(700, seed=5)
    cfg = akmc.Config(cells=(8, 8, 8), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32)
    with akmc.Simulation(cfg, np.zeros(2 * 8 ** 3, np.uint8), eps, E0, mlp) as sim:
        e_all = sim.eval_windows(w, akmc.PREC_FP32)
        perm = rng.permutation(len(w))
        e_perm = sim.eval_windows(w[perm], akmc.PREC_FP32)
        e_one = np.stack([sim.eval_windows(w[i:i + 1], akmc.PREC_FP32)[0] for i in range(0, len(w), 97)])
    assert np.array_equal(e_perm, e_all[perm])
    assert np.array_equal(e_one, e_all[::97])


def test_engine_matches_legacy_loop(akmc, orc, monkeypatch):
    """The phase engine and the grid-synchronous legacy inner loop (AKMC_LEGACY_LOOP=1) run the same FP64
    trajectory (both equal the oracle's)."""
    eps, E0 = _params()
    L = 32
    sp = synth.make_lattice((L, L, L), 1, synth.a508_atomic_fractions(), 50, seed=91)
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=3,
                      domain_cells=(8, 8, 8), window_s=synth.window_seconds(0.5, E0[0]))
    with akmc.Simulation(cfg, sp, eps, E0) as sim:
        sim.step(6)
        a = sim.state()
    monkeypatch.setenv("AKMC_LEGACY_LOOP", "1")
    with akmc.Simulation(cfg, sp, eps, E0) as sim:
        sim.step(6)
        b = sim.state()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    assert a[3]["events"] == b[3]["events"] and a[3]["hop_evals"] == b[3]["hop_evals"]
