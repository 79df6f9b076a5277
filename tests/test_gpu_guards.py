"""GPU tests of the range / capacity guards, the legacy-loop fallback for large sectors, the shared FP32
evaluator (engine == grid-synchronous loop, crowded domains) and checkpoint / resume through the C-ABI.

* Activation range: the FP32-equivalent evaluator splits activations into fp16 hi/lo.
  Power-of-two activation scales chosen at init from weight bounds keep every |h| * 2^-t <= 2^15, so weights
  with activations ~1e5 are evaluated within the 1e-5 rate bar instead of being silently clamped; with the
  scaling disabled (AKMC_NO_ACT_SCALE, fault injection) the clamp is counted and the call returns
  AKMC_ERR_RUNTIME instead of AKMC_OK.
* Capacity: a configuration whose sector can hold more vacancies than one engine CTA holds runs the
  grid-synchronous loop (any competing-set size) and stays bit-exact vs the oracle.
* Checkpoint / resume: lattice + slot-ordered vacancy sites + clocks + event counters +
  sweep counter resume a run bit-identically to the unsplit run (counter-based RNG: no RNG state).
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


def _rel(a, b):
    scale = np.maximum(np.abs(b), 1e-300)
    return np.where(b == 0.0, np.abs(a), np.abs(a - b) / scale)


def _big_activation_mlp():
    """Random network whose first four hidden units carry activations ~1e5 (b1 += 1e5); the matching W2
    rows are scaled by 1e-5 so the barriers stay O(1 eV)."""
    m = synth.random_mlp(seed=11).copy()
    o1 = 448 * 256
    m[o1:o1 + 4] += 1.0e5
    W2 = m[o1 + 256:o1 + 256 + 256 * 256].reshape(256, 256)
    W2[:4, :] *= 1.0e-5
    return m


def test_large_activations_meet_rate_bar(akmc, orc):
    mlp = _big_activation_mlp()
    wins = synth.random_windows(2000, seed=12)
    cfg = akmc.Config(cells=(8, 8, 8), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32)
    with akmc.Simulation(cfg, np.zeros(1024, np.uint8), mlp=mlp) as sim:
        E = sim.eval_windows(wins, akmc.PREC_FP32)
    ref = np.stack([orc.mlp_fp64(w, mlp) for w in wins])
    kT = cfg.kB * cfg.temperature_K
    rel = float(np.abs(np.expm1(-(E - ref) / kT)).max())
    assert rel <= RTOL_FAST, rel


def test_overflow_guard_returns_runtime_error(akmc, monkeypatch):
    """Fault injection: without the activation scales the fp16 clamp fires; eval_windows, rates and step
    return AKMC_ERR_RUNTIME (the counter used to be allocated but never read)."""
    monkeypatch.setenv("AKMC_NO_ACT_SCALE", "1")
    mlp = _big_activation_mlp()
    wins = synth.random_windows(300, seed=13)
    cfg = akmc.Config(cells=(8, 8, 8), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32)
    with akmc.Simulation(cfg, np.zeros(1024, np.uint8), mlp=mlp) as sim:
        with pytest.raises(akmc.AkmcError) as ei:
            sim.eval_windows(wins, akmc.PREC_FP32)
        assert ei.value.code == akmc.AKMC_ERR_RUNTIME
        E = sim.eval_windows(wins[:0], akmc.PREC_FP32)    # the counter was reset: the handle stays usable
        assert E.shape == (0, 8)
    L = 16
    eps, E0 = synth.illustrative_pair_params()
    sp = synth.make_lattice((L, L, L), 1, synth.a508_atomic_fractions(), 20, seed=3)
    cfg2 = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32, seed=3,
                       domain_cells=(8, 8, 8), window_s=synth.window_seconds(1.0, E0[0]))
    with akmc.Simulation(cfg2, sp, mlp=mlp) as sim:
        with pytest.raises(akmc.AkmcError) as ei:
            sim.step(1)
        assert ei.value.code == akmc.AKMC_ERR_RUNTIME
        with pytest.raises(akmc.AkmcError) as ei:
            sim.rates()
        assert ei.value.code == akmc.AKMC_ERR_RUNTIME


def _cluster(sp, L, center, half, n, rng):
    cx, cy, cz = center
    placed = 0
    while placed < n:
        x, y, z = (int(v) for v in rng.integers(0, half, size=3))
        b = int(rng.integers(0, 2))
        i = 2 * (((cx + x) % L) + L * (((cy + y) % L) + L * ((cz + z) % L))) + b
        if sp[i] != 6:
            sp[i] = 6
            placed += 1
    return sp


def test_large_sector_runs_bitexact(akmc, orc):
    """domain_cells 12^3 -> a sector of 6^3 cells (432 sites) can hold more vacancies than an engine CTA
    (256): the library runs the grid-synchronous loop.  300 vacancies packed into ONE sector (a competing
    set of 300, tree in scratch) plus a dilute background: bit-exact vs the oracle."""
    eps, E0 = synth.illustrative_pair_params()
    L = 36
    sp = synth.make_lattice((L, L, L), 1, synth.fe_cu_fractions(0.05), 60, seed=41)
    sp = _cluster(sp, L, (12, 12, 12), 6, 300, np.random.default_rng(42))
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=17,
                      domain_cells=(12, 12, 12), window_s=synth.window_seconds(0.5, E0[0]))
    ocfg = orc.Config(cells=cfg.cells, model=0, domain=cfg.domain_cells, window_s=cfg.window_s, seed=cfg.seed)
    st = orc.State.from_species(ocfg, sp)
    with akmc.Simulation(cfg, sp, eps, E0) as sim:
        c = sim.step(3)
        gsp, gvac, gclock, gctr = sim.state()
    orc.run(ocfg, st, 3, eps, E0)
    assert c["events"] > 50
    assert np.array_equal(gsp, st.species) and np.array_equal(gvac, st.vac) and np.array_equal(gclock, st.clock)
    assert gctr["events"] == st.counters[0] and gctr["hop_evals"] == st.counters[1]


@pytest.mark.parametrize("lam", [1.0, 0.25])
def test_fp32_engine_equals_grid_loop_crowded(akmc, orc, monkeypatch, lam):
    """FP32 tensor-core trajectories with crowded domains (multi-slot placement, > 16-member trees in scratch):
    the persistent phase engine and the grid-synchronous loop share the evaluator, so they must produce the
    same bits; the final rates meet the 1e-5 bar against the FP64 oracle and the composition is conserved."""
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=5)
    L = 32
    sp = synth.make_lattice((L, L, L), 1, synth.fe_cu_fractions(0.05), 100, seed=77)
    sp = _cluster(sp, L, (8, 8, 8), 4, 60, np.random.default_rng(78))      # 60 vacancies in one 4^3 sector
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32, seed=29,
                      domain_cells=(8, 8, 8), window_s=synth.window_seconds(lam, E0[0]))
    with akmc.Simulation(cfg, sp, mlp=mlp) as sim:
        sim.step(4)
        a = sim.state()
        G, _ = sim.rates()
    monkeypatch.setenv("AKMC_LEGACY_LOOP", "1")
    with akmc.Simulation(cfg, sp, mlp=mlp) as sim:
        sim.step(4)
        b = sim.state()
    assert a[3]["events"] > 50
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    assert a[3]["events"] == b[3]["events"] and a[3]["hop_evals"] == b[3]["hop_evals"]
    assert np.array_equal(np.bincount(a[0], minlength=7), np.bincount(sp, minlength=7))
    ocfg = orc.Config(cells=cfg.cells, model=1, domain=cfg.domain_cells, window_s=cfg.window_s, seed=cfg.seed)
    Go, _ = orc.rates(ocfg, a[0], a[1], mlp=mlp)
    assert np.array_equal(G == 0.0, Go == 0.0)
    assert float(_rel(G, Go).max()) <= RTOL_FAST


def _split_vs_unsplit(akmc, cfg, sp, n1, n2, eps=None, E0=None, mlp=None):
    with akmc.Simulation(cfg, sp, eps, E0, mlp) as sim:
        sim.step(n1 + n2)
        full = sim.state()
    with akmc.Simulation(cfg, sp, eps, E0, mlp) as sim:
        sim.step(n1)
        csp, cvac, cclock, _ = sim.state()
        nev, sweep = sim.progress()
    with akmc.Simulation(cfg, csp, eps, E0, mlp) as sim:       # a fresh handle from the checkpointed lattice
        sim.restore(cvac, cclock, nev, sweep)
        sim.step(n2)
        resumed = sim.state()
    return full, resumed


def test_checkpoint_resume_serial_voxels(akmc, orc):
    """Serial BKL in 6 voxels, FP64 pair: run 300 + 700 events == 1000 events == the oracle."""
    eps, E0 = synth.illustrative_pair_params()
    L = 16
    sp = synth.make_lattice((L, L, L), 6, synth.a508_atomic_fractions(), 5, seed=19)
    cfg = akmc.Config(cells=(L, L, L), n_voxels=6, barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=8)
    full, resumed = _split_vs_unsplit(akmc, cfg, sp, 300, 700, eps, E0)
    for x, y in zip(full[:3], resumed[:3]):
        assert np.array_equal(x, y)
    ocfg = orc.Config(cells=cfg.cells, n_voxels=6, model=0, seed=cfg.seed)
    st = orc.State.from_species(ocfg, sp)
    orc.run(ocfg, st, 1000, eps, E0)
    assert np.array_equal(resumed[0], st.species) and np.array_equal(resumed[1], st.vac)
    assert np.array_equal(resumed[2], st.clock)


@pytest.mark.parametrize("model", ["pair", "mlp"])
def test_checkpoint_resume_sublattice(akmc, model):
    """Sublattice sweeps (FP64 pair / FP32 tensor-core MLP): 3 + 4 sweeps == 7 sweeps bit for bit, including
    the sector permutation and phase counters of the resumed sweeps."""
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=6) if model == "mlp" else None
    L = 32
    sp = synth.make_lattice((L, L, L), 1, synth.a508_atomic_fractions(), 60, seed=23)
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_MLP if mlp is not None else akmc.MODEL_PAIR,
                      precision=akmc.PREC_FP32 if mlp is not None else akmc.PREC_FP64, seed=31,
                      domain_cells=(8, 8, 8), window_s=synth.window_seconds(1.0, E0[0]))
    full, resumed = _split_vs_unsplit(akmc, cfg, sp, 3, 4, eps, E0, mlp)
    for x, y in zip(full[:3], resumed[:3]):
        assert np.array_equal(x, y)
    assert full[3]["events"] > 50


def test_restore_rejects_bad_checkpoints(akmc):
    eps, E0 = synth.illustrative_pair_params()
    L = 16
    sp = synth.make_lattice((L, L, L), 2, synth.a508_atomic_fractions(), 4, seed=2)
    cfg = akmc.Config(cells=(L, L, L), n_voxels=2, barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=8)
    with akmc.Simulation(cfg, sp, eps, E0) as sim:
        _, vac, clock, _ = sim.state()
        nev, sweep = sim.progress()
        bad = vac.copy(); bad[0] = bad[0] + 1 if sp[bad[0] + 1] != 6 else bad[0] + 2    # not a vacancy site
        for args in [(bad, clock, nev, 0), (vac[::-1].copy(), clock, nev, 0), (vac, -clock - 1.0, nev, 0),
                     (vac, clock, nev - 5, 0), (vac, clock, nev, -1)]:
            with pytest.raises(akmc.AkmcError) as ei:
                sim.restore(*args)
            assert ei.value.code == akmc.AKMC_ERR_INVALID
        sim.restore(vac, clock, nev, sweep)                  # the real checkpoint is accepted


# ----------------------------------------------------------------------------- bulk evaluator (akmc_bulk.cu)
@pytest.mark.parametrize("weights,prec", [("physics", "fp32"), ("random", "fp32"), ("physics", "fast")])
def test_bulk_evaluator_bitexact_vs_cluster_evaluator(akmc, monkeypatch, weights, prec):
    """The warp-specialised bulk evaluator and the phase engine's cluster evaluator (AKMC_EVAL_ENGINE=1) give
    the same bits for every window (ragged last tile: 3000 = 23 x 128 + 56 rows), FP32-equivalent and FP16-fast:
    one arithmetic for every path that forms a rate (R7)."""
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=4) if weights == "physics" else synth.random_mlp(seed=9)
    P = akmc.PREC_FP32 if prec == "fp32" else akmc.PREC_FP16_FAST
    wins = synth.random_windows(3000, seed=21)
    cfg = akmc.Config(cells=(8, 8, 8), barrier_model=akmc.MODEL_MLP, precision=P)
    with akmc.Simulation(cfg, np.zeros(1024, np.uint8), mlp=mlp) as sim:
        e_bulk = sim.eval_windows(wins, P)
    monkeypatch.setenv("AKMC_EVAL_ENGINE", "1")
    with akmc.Simulation(cfg, np.zeros(1024, np.uint8), mlp=mlp) as sim:
        e_eng = sim.eval_windows(wins, P)
    assert np.array_equal(e_bulk.view(np.uint64), e_eng.view(np.uint64))


def test_bulk_rates_lattice_bitexact_and_within_bar(akmc, orc, monkeypatch):
    """akmc_rates on a 64^3 RPV voxel with 300 vacancies: bulk == cluster evaluator bit for bit, and within the
    1e-5 bar of the FP64 oracle with exact masks."""
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=2)
    L = 64
    sp = synth.make_lattice((L, L, L), 1, synth.a508_atomic_fractions(), 300, seed=31)
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32)
    with akmc.Simulation(cfg, sp, mlp=mlp) as sim:
        G1, E1 = sim.rates()
        _, vac, _, _ = sim.state(species=False)
    monkeypatch.setenv("AKMC_EVAL_ENGINE", "1")
    with akmc.Simulation(cfg, sp, mlp=mlp) as sim:
        G2, E2 = sim.rates()
    assert np.array_equal(G1.view(np.uint64), G2.view(np.uint64)) and np.array_equal(E1.view(np.uint64), E2.view(np.uint64))
    ocfg = orc.Config(cells=cfg.cells, model=1)
    Go, _ = orc.rates(ocfg, sp, vac, mlp=mlp)
    assert np.array_equal(G1 == 0.0, Go == 0.0)
    assert float(_rel(G1, Go).max()) <= RTOL_FAST


# ----------------------------------------------------------------------------- dynamic voxel scheduling (Eq. 10)
def _eq10_order(sp, cells, nvox, E0, T, kB=8.617333262e-5):
    S = 2 * cells[0] * cells[1] * cells[2]
    W = []
    for v in range(nvox):
        c = np.bincount(sp[v * S:(v + 1) * S], minlength=7)
        n = c[:6].sum()
        Ev = float((c[:6] * np.asarray(E0)[:6]).sum() / n)
        W.append(8.0 * c[6] * np.exp(-Ev / (kB * T[v])))
    return np.array(sorted(range(nvox), key=lambda v: -W[v]), dtype=np.int32)   # stable on ties


def test_voxel_dispatch_order_is_eq10(akmc):
    """P:481-490 / S:658-670: voxels are dispatched in descending W_v = 8 m_v exp(-E_v / kB T_v) (E_v = the
    composition-weighted mean E0), recomputed when the voxel temperatures change; ties keep voxel order."""
    eps, E0 = synth.illustrative_pair_params()
    L, nvox = 8, 40
    rng = np.random.default_rng(4)
    parts = [synth.make_lattice((L, L, L), 1, synth.fe_cu_fractions(float(rng.uniform(0.0, 0.3))),
                                int(rng.integers(1, 6)), seed=100 + v) for v in range(nvox)]
    sp = np.concatenate(parts)
    cfg = akmc.Config(cells=(L, L, L), n_voxels=nvox, barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64)
    with akmc.Simulation(cfg, sp, eps, E0) as sim:
        assert np.array_equal(sim.voxel_order(), _eq10_order(sp, (L, L, L), nvox, E0, [563.0] * nvox))
        T = synth.voxel_temperatures(nvox, seed=3)
        sim.set_voxel_temperatures(T)
        assert np.array_equal(sim.voxel_order(), _eq10_order(sp, (L, L, L), nvox, E0, T))


# ----------------------------------------------------------------------------- dataflow sweeps (f1)
def _df_pair(akmc, cfg, sp, sweeps, eps=None, E0=None, mlp=None):
    with akmc.Simulation(cfg, sp, eps, E0, mlp) as sim:
        sim.step(sweeps)
        sync = sim.state()
    with akmc.Simulation(cfg, sp, eps, E0, mlp) as sim:
        sim.set_dataflow(True)
        half = sweeps // 2
        sim.step(half)
        sim.step(sweeps - half)
        df = sim.state()
    return sync, df


@pytest.mark.parametrize("cells,domain,lam", [((32, 32, 32), (8, 8, 8), 1.0), ((48, 32, 40), (8, 8, 8), 0.25),
                                              ((18, 24, 30), (6, 8, 10), 1.0)])
def test_dataflow_sweep_bitexact_fp64(akmc, orc, cells, domain, lam):
    """P:405-418 readiness signals (f1): tiles start a phase when the 27 tiles around them finished the previous
    one; the FP64 trajectory equals the phase-synchronous one and the oracle's, bit for bit (anisotropic
    geometry and ragged tiles included)."""
    eps, E0 = synth.illustrative_pair_params()
    sp = synth.make_lattice(cells, 1, synth.a508_atomic_fractions(), 80, seed=61)
    cfg = akmc.Config(cells=cells, barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=7,
                      domain_cells=domain, window_s=synth.window_seconds(lam, E0[0]))
    sync, df = _df_pair(akmc, cfg, sp, 6, eps, E0)
    assert df[3]["events"] > 50
    for x, y in zip(sync[:3], df[:3]):
        assert np.array_equal(x, y)
    assert df[3]["events"] == sync[3]["events"] and df[3]["hop_evals"] == sync[3]["hop_evals"]
    ocfg = orc.Config(cells=cells, model=0, domain=domain, window_s=cfg.window_s, seed=cfg.seed)
    st = orc.State.from_species(ocfg, sp)
    orc.run(ocfg, st, 6, eps, E0)
    assert np.array_equal(df[0], st.species) and np.array_equal(df[1], st.vac) and np.array_equal(df[2], st.clock)


def test_dataflow_sweep_fp32_crowded(akmc):
    """FP32 tensor-core engine, crowded domains (multi-slot, > 16-member trees): dataflow == synchronous bits."""
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.physics_mlp(eps, E0, residual=0.02, seed=5)
    L = 32
    sp = synth.make_lattice((L, L, L), 1, synth.fe_cu_fractions(0.05), 100, seed=77)
    sp = _cluster(sp, L, (8, 8, 8), 4, 60, np.random.default_rng(78))
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32, seed=29,
                      domain_cells=(8, 8, 8), window_s=synth.window_seconds(1.0, E0[0]))
    sync, df = _df_pair(akmc, cfg, sp, 6, mlp=mlp)
    assert df[3]["events"] > 50
    for x, y in zip(sync[:3], df[:3]):
        assert np.array_equal(x, y)


def test_dataflow_sweep_crowded_tile_bitexact(akmc, orc):
    """A tile-phase with more than 64 vacancies (90 packed into one 4^3-cell sector): the general activation
    path; FP64 dataflow == synchronous == oracle."""
    eps, E0 = synth.illustrative_pair_params()
    L = 32
    sp = synth.make_lattice((L, L, L), 1, synth.fe_cu_fractions(0.05), 80, seed=91)
    sp = _cluster(sp, L, (16, 16, 16), 4, 90, np.random.default_rng(92))
    cfg = akmc.Config(cells=(L, L, L), barrier_model=akmc.MODEL_PAIR, precision=akmc.PREC_FP64, seed=5,
                      domain_cells=(8, 8, 8), window_s=synth.window_seconds(1.0, E0[0]))
    sync, df = _df_pair(akmc, cfg, sp, 4, eps, E0)
    for x, y in zip(sync[:3], df[:3]):
        assert np.array_equal(x, y)
    ocfg = orc.Config(cells=(L, L, L), model=0, domain=(8, 8, 8), window_s=cfg.window_s, seed=cfg.seed)
    st = orc.State.from_species(ocfg, sp)
    orc.run(ocfg, st, 4, eps, E0)
    assert np.array_equal(df[0], st.species) and np.array_equal(df[1], st.vac)
