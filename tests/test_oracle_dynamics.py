"""Dynamics pins of the oracle (serial BKL and windowed sublattice), -m "not gpu".

Closed forms and statistics the paper/SPEC fix: conservation, residence time
Exp(1) with mean 1/Gamma_tot, selection law Gamma_a/Gamma_tot (S:202,
P:294-298 Eq. 2), Boltzmann stationarity by exact enumeration (north star),
sublattice sector independence (reading A20) and degenerate cases.
"""
import math

import numpy as np
import pytest

import synth


def _pure_fe_with_vacancy(L, v_cell=(2, 2, 2)):
    sp = np.zeros(2 * L ** 3, dtype=np.uint8)
    v = 2 * (v_cell[0] + L * (v_cell[1] + L * v_cell[2]))
    sp[v] = 6
    return sp, v


def test_conservation_and_vacancy_registry(orc):
    """S:84 composition conservation; S:38 vacancy list == occupancy, after many events."""
    L = 8
    fr = synth.a508_atomic_fractions()
    sp = synth.make_lattice((L, L, L), 2, fr, 3, seed=5)
    cfg = orc.Config(cells=(L, L, L), n_voxels=2, model=0, seed=9)
    eps, E0 = synth.illustrative_pair_params()
    st = orc.State.from_species(cfg, sp)
    counts0 = np.bincount(sp, minlength=7)
    rc = orc.run(cfg, st, 500, eps, E0)
    assert rc == orc.ORC_OK
    assert np.array_equal(np.bincount(st.species, minlength=7), counts0)
    assert np.array_equal(np.sort(st.vac), np.flatnonzero(st.species == 6))
    assert st.counters[0] == 1000 and np.all(st.nev == 500)
    # vacancies never leave their voxel
    n = cfg.sites_per_voxel
    assert np.array_equal(np.sort(st.vac // n), np.repeat([0, 1], 3))


def test_reversal_identity(orc):
    """apply then apply the reverse hop restores the occupancy bit-exactly.  We use the
    event the oracle selects, then undo it by swapping back and compare."""
    L = 6
    sp = synth.make_lattice((L, L, L), 1, synth.fe_cu_fractions(0.2), 2, seed=1)
    cfg = orc.Config(cells=(L, L, L), model=0, seed=4)
    eps, E0 = synth.illustrative_pair_params()
    st = orc.State.from_species(cfg, sp)
    before = st.copy()
    orc.run(cfg, st, 1, eps, E0)
    moved = np.flatnonzero(st.vac != before.vac)
    assert moved.size == 1
    i = moved[0]
    a, b = before.vac[i], st.vac[i]
    undo = st.species.copy(); undo[a], undo[b] = undo[b], undo[a]
    assert np.array_equal(undo, before.species)


def test_residence_time_exponential(orc):
    """dt * Gamma_tot ~ iid Exp(1); pure Fe: Gamma_tot = 8 nu0 e^{-E0/kT}."""
    from scipy import stats
    L = 6
    sp, v = _pure_fe_with_vacancy(L)
    eps, E0 = synth.illustrative_pair_params()
    cfg = orc.Config(cells=(L, L, L), model=0, seed=123)
    st = orc.State.from_species(cfg, sp)
    gtot = 8 * cfg.nu0 * math.exp(-E0[0] / (cfg.kB * cfg.T))
    xs = []
    for _ in range(4000):
        c0 = st.clock[0]
        orc.run(cfg, st, 1, eps, E0)
        xs.append((st.clock[0] - c0) * gtot)
    xs = np.array(xs)
    assert stats.kstest(xs, "expon").pvalue > 1e-3
    assert abs(xs.mean() - 1.0) < 4.0 / math.sqrt(xs.size)


def test_selection_law(orc):
    """S:202 / Eq. 2: hop k is chosen with probability Gamma_k / Gamma_tot (chi^2 over seeds).
    Rates from orc.barriers (pinned separately); the selection tree/descent is under test."""
    from scipy import stats
    L = 6
    sp, v = _pure_fe_with_vacancy(L)
    # solute neighbours make the 8 rates unequal
    w = orc.window_offsets()
    cfg = orc.Config(cells=(L, L, L), model=0)
    eps, E0 = synth.illustrative_pair_params()
    rng = np.random.default_rng(0)
    for j in range(8, 40):
        if rng.random() < 0.5:
            p = np.array([4 + w[j, 0] + 0, 4 + w[j, 1], 4 + w[j, 2]]) % (2 * L)
            sp[2 * ((p[0] >> 1) + L * ((p[1] >> 1) + L * (p[2] >> 1))) + (p[0] & 1)] = rng.integers(1, 6)
    for k in (1, 4):
        p = np.array([4 + w[k, 0], 4 + w[k, 1], 4 + w[k, 2]]) % (2 * L)
        sp[2 * ((p[0] >> 1) + L * ((p[1] >> 1) + L * (p[2] >> 1))) + (p[0] & 1)] = 1
    E, G, _ = orc.barriers(cfg, sp, v, eps, E0)
    prob = G / G.sum()
    n = 6000
    counts = np.zeros(8)
    for seed in range(n):
        cfg.seed = seed
        st = orc.State.from_species(cfg, sp)
        orc.run(cfg, st, 1, eps, E0)
        dv = st.vac[0]
        for k in range(8):
            p = np.array([4 + w[k, 0], 4 + w[k, 1], 4 + w[k, 2]]) % (2 * L)
            if 2 * ((p[0] >> 1) + L * ((p[1] >> 1) + L * (p[2] >> 1))) + (p[0] & 1) == dv:
                counts[k] += 1
    assert counts.sum() == n
    assert stats.chisquare(counts, prob * n).pvalue > 1e-3


def test_terminal_no_vacancy(orc):
    """no vacancies -> terminal signal, state unchanged."""
    L = 4
    cfg = orc.Config(cells=(L, L, L), model=0)
    eps, E0 = synth.illustrative_pair_params()
    st = orc.State.from_species(cfg, np.zeros(2 * L ** 3, dtype=np.uint8))
    assert orc.run(cfg, st, 3, eps, E0) == orc.ORC_TERMINAL
    assert st.counters[0] == 0 and st.clock[0] == 0.0


def _bcc_pos(i, L):
    b = i & 1; c = i >> 1
    return np.array([2 * (c % L) + b, 2 * ((c // L) % L) + b, 2 * (c // (L * L)) + b])


def _is_1nn(a, b, L):
    d = (_bcc_pos(a, L) - _bcc_pos(b, L)) % (2 * L)
    d = np.minimum(d, 2 * L - d)
    return bool(np.all(d == 1))


def test_zero_rate_vacancy_never_selected(orc):
    """Degenerate case of the method: a vacancy whose eight first neighbours are all vacancies has every
    hop masked (m_k = 0; Gamma = 0 exactly, A14), so its leaf R_i = 0 lies inside the competing
    set.  Pins: brute-force geometry (the eight sites at half-cell distance (1,1,1) are V), all eight rates
    of that vacancy are exactly 0 while its neighbours have positive rates, and over 300 seeds the first
    BKL event never moves it and always takes a hop of positive rate."""
    L = 8
    eps, E0 = synth.illustrative_pair_params()
    base = synth.make_lattice((L, L, L), 1, synth.fe_cu_fractions(0.05), 2, seed=5)
    sp, c = synth.with_vacancy_cluster(base, (L, L, L), (4, 4, 4))
    nn = [j for j in range(sp.size) if _is_1nn(c, j, L)]
    assert len(nn) == 8 and all(sp[j] == 6 for j in nn)
    cfg = orc.Config(cells=(L, L, L), model=0)
    st0 = orc.State.from_species(cfg, sp)
    R, _ = orc.rates(cfg, st0.species, st0.vac, eps, E0)
    ic = int(np.flatnonzero(st0.vac == c)[0])
    assert np.all(R[ic] == 0.0)
    assert all(R[int(np.flatnonzero(st0.vac == j)[0])].sum() > 0 for j in nn)
    for seed in range(300):
        cfg = orc.Config(cells=(L, L, L), model=0, seed=seed)
        st = st0.copy()
        assert orc.run(cfg, st, 1, eps, E0) == 0
        moved = np.flatnonzero(st.vac != st0.vac)
        assert moved.size == 1 and int(moved[0]) != ic
        i = int(moved[0])
        assert _is_1nn(int(st0.vac[i]), int(st.vac[i]), L)
        d = (_bcc_pos(int(st.vac[i]), L) - _bcc_pos(int(st0.vac[i]), L)) % (2 * L)   # +1 or 2L-1 per axis
        k = 4 * (d[0] == 1) + 2 * (d[1] == 1) + (d[2] == 1)                           # A4: k = 4[hx>0]+2[hy>0]+[hz>0]
        assert R[i, k] > 0


@pytest.mark.slow
def test_boltzmann_stationarity_enumeration(orc):
    """North star / SURVEY 8(c): Boltzmann stationary distribution by exact enumeration on a tiny
    lattice.  L = 4 (128 sites), 1 V + 2 Cu in Fe; the 8,001 translation classes (V fixed at site 0)
    get pi ~ exp(-E/kT) from the FULL bond-count energy; a long serial BKL run weighted by the mean
    residence time 1/Gamma_tot matches <#V-Cu 1NN> and <#Cu-Cu 1NN> within 4 sigma (batch means)."""
    L = 4
    n = 2 * L ** 3
    eps = np.zeros((2, 7, 7))
    eps[0] = -0.78; eps[1] = -0.39
    eps[0, 1, 1] = -0.95; eps[0, 1, 0] = eps[0, 0, 1] = -0.76      # Cu-Cu attraction
    eps[0, 6, :] = eps[0, :, 6] = -0.20; eps[0, 6, 1] = eps[0, 1, 6] = -0.33   # V-Cu binding
    eps[1, 6, :] = eps[1, :, 6] = -0.10
    E0 = np.array([0.62, 0.54, 0.68, 0.60, 0.78, 0.70, 0.0])
    cfg = orc.Config(cells=(L, L, L), model=0, T=900.0, seed=77)
    kT = cfg.kB * cfg.T
    nn = np.array([[_is_1nn(a, b, L) for b in range(n)] for a in range(n)])
    # exact expectation over classes (V at 0, Cu at {i < j} among 1..127)
    Es, o1, o2 = [], [], []
    base = np.zeros(n, dtype=np.uint8); base[0] = 6
    for i in range(1, n):
        for j in range(i + 1, n):
            sp = base.copy(); sp[i] = 1; sp[j] = 1
            Es.append(orc.system_energy(cfg, sp, 0, eps))
            o1.append(int(nn[0, i]) + int(nn[0, j]))
            o2.append(int(nn[i, j]))
    Es = np.array(Es); o1 = np.array(o1); o2 = np.array(o2)
    w = np.exp(-(Es - Es.min()) / kT); w /= w.sum()
    exact1, exact2 = (w * o1).sum(), (w * o2).sum()
    # clamp-free check for this parameter set (detailed balance needs no clamping)
    # dynamics: long serial run, mean-residence-time weighting
    sp = base.copy(); sp[5] = 1; sp[77] = 1
    st = orc.State.from_species(cfg, sp)
    nev = 120000
    obs1 = np.empty(nev); obs2 = np.empty(nev); wt = np.empty(nev)
    for e in range(nev):
        R, _ = orc.rates(cfg, st.species, st.vac, eps, E0)
        v = st.vac[0]
        cu = np.flatnonzero(st.species == 1)
        obs1[e] = int(nn[v, cu[0]]) + int(nn[v, cu[1]])
        obs2[e] = int(nn[cu[0], cu[1]])
        wt[e] = 1.0 / R.sum()
        orc.run(cfg, st, 1, eps, E0)
    assert st.counters[3] == 0
    burn = 2000
    for obs, exact in ((obs1, exact1), (obs2, exact2)):
        o = obs[burn:]; ww = wt[burn:]
        est = (o * ww).sum() / ww.sum()
        nb = 40
        bs = np.array_split(np.arange(o.size), nb)
        bm = np.array([(o[b] * ww[b]).sum() / ww[b].sum() for b in bs])
        sigma = bm.std(ddof=1) / math.sqrt(nb)
        print("boltzmann", est, exact, sigma)
        assert abs(est - exact) < 4 * sigma + 1e-3, (est, exact, sigma)


def test_sublattice_strict_equals_bucketed(orc):
    """Reading A20: domains never interact inside a phase (sector >= 3 cells), so building each
    domain's active set once per phase (bucketed) equals re-scanning all vacancies (strict)."""
    L = 16
    fr = synth.fe_cu_fractions(0.05)
    sp = synth.make_lattice((L, L, L), 1, fr, 40, seed=3)
    eps, E0 = synth.illustrative_pair_params()
    win = synth.window_seconds(1.0, E0[0])
    res = []
    for strict in (0, 1):
        cfg = orc.Config(cells=(L, L, L), model=0, domain=(8, 8, 8), window_s=win, seed=21, strict=strict)
        st = orc.State.from_species(cfg, sp)
        orc.run(cfg, st, 6, eps, E0)
        res.append(st)
    assert np.array_equal(res[0].species, res[1].species)
    assert np.array_equal(res[0].vac, res[1].vac)
    assert np.array_equal(res[0].counters, res[1].counters)
    assert res[0].counters[0] > 50                       # events happened
    assert res[0].clock[0] == pytest.approx(6 * win)     # clock += window per sweep


def test_sector_permutation_is_permutation(orc):
    """A19: the per-sweep sector order is a permutation of the 8 octants, varying with the sweep."""
    perms = [tuple(orc.sector_perm(99, s)) for s in range(50)]
    for p in perms:
        assert sorted(p) == list(range(8))
    assert len(set(perms)) > 30


def test_per_voxel_temperature(orc):
    """C4 variant: each voxel's rates follow Eq. 8 at ITS temperature.
    Pure-Fe voxels with one vacancy: every rate = nu0 exp(-E0[Fe]/(kB T_v)) and the mean
    residence time of voxel v is 1/(8 nu0 exp(-E0/kB T_v)); voxels are independent."""
    L = 6
    nvox = 3
    one, v = _pure_fe_with_vacancy(L)
    sp = np.concatenate([one] * nvox)
    eps, E0 = synth.illustrative_pair_params()
    T = np.array([450.0, 563.0, 700.0])
    cfg = orc.Config(cells=(L, L, L), n_voxels=nvox, model=0, seed=41, voxel_T=T)
    st = orc.State.from_species(cfg, sp)
    R, E = orc.rates(cfg, st.species, st.vac, eps, E0)
    for i in range(nvox):
        g = cfg.nu0 * math.exp(-E0[0] / (cfg.kB * T[i]))
        assert np.allclose(R[i], g, rtol=1e-14, atol=0.0), (i, R[i], g)
    # uniform T through voxel_T == the scalar path, bit for bit
    cu = orc.Config(cells=(L, L, L), n_voxels=nvox, model=0, seed=41, T=563.0)
    cv = orc.Config(cells=(L, L, L), n_voxels=nvox, model=0, seed=41, voxel_T=np.full(nvox, 563.0))
    assert np.array_equal(orc.rates(cu, sp, st.vac, eps, E0)[0], orc.rates(cv, sp, st.vac, eps, E0)[0])
    n = 3000
    orc.run(cfg, st, n, eps, E0)
    for i in range(nvox):
        gtot = 8 * cfg.nu0 * math.exp(-E0[0] / (cfg.kB * T[i]))
        mean = st.clock[i] / n * gtot                 # mean of Exp(1) draws
        assert abs(mean - 1.0) < 5.0 / math.sqrt(n), (i, mean)


def test_run_until_horizon(orc):
    """Voxel-ensemble mode: horizons split a run without changing it, and no voxel clock passes
    the horizon."""
    L = 8
    nvox = 3
    sp = synth.make_lattice((L, L, L), nvox, synth.a508_atomic_fractions(), 4, seed=17)
    eps, E0 = synth.illustrative_pair_params()
    cfg = orc.Config(cells=(L, L, L), n_voxels=nvox, model=0, seed=23)
    t1, t2 = 8e-8, 2e-7                # ~ 40 / 100 events per voxel (Gamma_tot ~ 5e8 /s)
    a = orc.State.from_species(cfg, sp)
    orc.run_until(cfg, a, t2, 10 ** 6, eps, E0)
    b = orc.State.from_species(cfg, sp)
    orc.run_until(cfg, b, t1, 10 ** 6, eps, E0)
    orc.run_until(cfg, b, t2, 10 ** 6, eps, E0)
    for f in ("species", "vac", "clock", "nev"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.counters[0] == b.counters[0] > 20
    assert np.all(a.clock <= t2)


def test_run_until_single_voxel_bruteforce(orc):
    """One voxel: run_until(t) stops exactly before the first event with time > t (S:198 clock)."""
    L = 8
    sp = synth.make_lattice((L, L, L), 1, synth.fe_cu_fractions(0.03), 2, seed=19)
    eps, E0 = synth.illustrative_pair_params()
    cfg = orc.Config(cells=(L, L, L), model=0, seed=29)
    t = 2e-7
    a = orc.State.from_species(cfg, sp)
    orc.run_until(cfg, a, t, 10 ** 6, eps, E0)
    ref = orc.State.from_species(cfg, sp)
    n = 0
    while True:
        trial = ref.copy()
        orc.run(cfg, trial, 1, eps, E0)
        if trial.clock[0] > t:
            break
        ref = trial
        n += 1
    assert n > 10 and a.nev[0] == n
    for f in ("species", "vac", "clock", "nev"):
        assert np.array_equal(getattr(a, f), getattr(ref, f)), f


def test_run_until_poisson_counts(orc):
    """Pure Fe, one vacancy per voxel: Gamma_tot = 8 nu0 e^{-E0/kT} is constant, so the number of events
    by time t is Poisson(Gamma_tot t); mean over 200 voxels within 4 sigma."""
    L = 6
    nvox = 200
    one, _ = _pure_fe_with_vacancy(L)
    sp = np.concatenate([one] * nvox)
    eps, E0 = synth.illustrative_pair_params()
    cfg = orc.Config(cells=(L, L, L), n_voxels=nvox, model=0, seed=31)
    gtot = 8 * cfg.nu0 * math.exp(-E0[0] / (cfg.kB * cfg.T))
    lam = 12.0
    st = orc.State.from_species(cfg, sp)
    orc.run_until(cfg, st, lam / gtot, 10 ** 6, eps, E0)
    n = st.nev.astype(float)
    assert abs(n.mean() - lam) < 4.0 * math.sqrt(lam / nvox), n.mean()
    assert abs(n.var() / lam - 1.0) < 0.35


def _unwrap_step(p0, p1, L):
    """half-cell displacement of one 1NN hop under the periodic box of L cells (|component| = 1)"""
    d = (p1 - p0 + L) % (2 * L) - L
    return d


def _half_cell_pos(site, L):
    cell, b = site // 2, site % 2
    x = cell % L; y = (cell // L) % L; z = cell // (L * L)
    return np.stack([2 * x + b, 2 * y + b, 2 * z + b], axis=-1)


def test_pure_fe_vacancy_diffusivity(orc):
    """in pure Fe a vacancy random-walks on the bcc 1NN vectors (a/2)(+-1,+-1,+-1) with 8 equal rates
    Gamma, so D = (1/6) sum_k Gamma |d_k|^2 = Gamma a^2: after n hops E|R|^2 = n (3/4) a^2 and E t = n/(8 Gamma),
    i.e. E|R|^2 / (6 E t) = Gamma a^2.  200 independent voxels, 150 hops each."""
    L = 6
    nvox, n = 200, 150
    one, _ = _pure_fe_with_vacancy(L)
    sp = np.concatenate([one] * nvox)
    eps, E0 = synth.illustrative_pair_params()
    cfg = orc.Config(cells=(L, L, L), n_voxels=nvox, model=0, seed=37)
    st = orc.State.from_species(cfg, sp)
    spv = 2 * L ** 3
    pos = _half_cell_pos(st.vac - np.arange(nvox) * spv, L)
    R = np.zeros((nvox, 3))
    for _ in range(n):
        orc.run(cfg, st, 1, eps, E0)
        p1 = _half_cell_pos(st.vac - np.arange(nvox) * spv, L)
        d = _unwrap_step(pos, p1, L)
        assert np.all(np.abs(d) == 1)                   # every hop is a 1NN vector (1/2,1/2,1/2) cell
        R += d
        pos = p1
    a = 1.0                                             # lengths in cells: one half-cell unit = a/2
    msd = np.mean(np.sum((R * a / 2) ** 2, axis=1))
    gamma = cfg.nu0 * math.exp(-E0[0] / (cfg.kB * cfg.T))
    D_est = msd / (6.0 * st.clock.mean())
    # |R|^2 has mean n*3/4 and sd ~ n*3/4*sqrt(2/3); the clock mean is n/(8 Gamma) with relative sd 1/sqrt(n nvox)
    rel_sd = math.sqrt(2.0 / 3.0) / math.sqrt(nvox) + 1.0 / math.sqrt(n * nvox)
    assert abs(D_est / (gamma * a * a) - 1.0) < 4.0 * rel_sd, (D_est, gamma)


def test_sublattice_time_consistency(orc):
    """Windowed synchronous sublattice (A19): with configuration-independent rates (all pair
    energies equal -> dE = 0) every isolated vacancy hops at Gamma_tot = 8 nu0 e^{-E0/kT} in serial
    BKL.  A sweep advances the clock by the window and runs each vacancy in its sector's phase, so
    events / (vacancies x Gamma_tot x clock) -> 1 as lambda -> 0, with the O(lambda) deficit of vacancies
    that leave their sector mid-window (-0.34 % at lambda = 1/4, -3.7 % at lambda = 1)."""
    L = 48
    eps, E0 = synth.illustrative_pair_params()
    eps = np.full_like(eps, -0.5)
    sp = np.zeros(2 * L ** 3, dtype=np.uint8)
    cells = [(x, y, z) for x in range(1, L, 8) for y in range(1, L, 8) for z in range(1, L, 8)]
    for (x, y, z) in cells:                             # one vacancy per 8^3 domain, 8 cells apart
        sp[2 * (x + L * (y + L * z))] = 6
    nvac = len(cells)
    gtot = 8 * 6.0e12 * math.exp(-E0[0] / (8.617333262e-5 * 563.0))
    ratio = {}
    for lam, sweeps in ((0.25, 200), (1.0, 60)):
        cfg = orc.Config(cells=(L, L, L), model=0, domain=(8, 8, 8), window_s=synth.window_seconds(lam, E0[0]),
                         seed=43)
        st = orc.State.from_species(cfg, sp)
        orc.run(cfg, st, sweeps, eps, E0)
        assert st.clock[0] == pytest.approx(sweeps * cfg.window_s, rel=1e-12)
        expected = nvac * gtot * st.clock[0]
        ratio[lam] = (float(st.counters[0]) / expected, 1.0 / math.sqrt(expected))
    r, sd = ratio[0.25]
    assert abs(r - 1.0) < 4.0 * sd + 0.005, ratio
    r1, sd1 = ratio[1.0]
    assert r1 < 1.0 and abs(r1 - (1.0 - 0.037)) < 4.0 * sd1, ratio


def test_mfpt_poisson_equation(orc):
    """P:338-347 (Eq. 5, Dynkin): the mean first-passage time tau(s) to an absorbing set solves
    sum_a Gamma_a(s) [tau(Phi(s,a)) - tau(s)] + 1 = 0.  Enumerable space: L = 4 (128 sites), 1 V + 1 Cu in Fe,
    absorbing = V and Cu first neighbours.  tau from the sparse linear solve over all 16,256 (V, Cu) states
    (rates from the oracle's barriers) must equal the mean absorption time of serial BKL episodes
    (S:195-198 clock) within 4 standard errors; with it, Eq. 7 with the exact u = Gamma_tot tau gives
    delta-tau = tau(s) - tau(s') on every transition (plug-in identity)."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.linalg import spsolve
    L = 4
    n = 2 * L ** 3
    eps = np.zeros((2, 7, 7))
    eps[0] = -0.78; eps[1] = -0.39
    eps[0, 6, :] = eps[0, :, 6] = -0.20; eps[0, 6, 1] = eps[0, 1, 6] = -0.33
    eps[1, 6, :] = eps[1, :, 6] = -0.10; eps[1, 6, 1] = eps[1, 1, 6] = -0.18   # V-Cu 2NN binding
    E0 = np.array([0.62, 0.54, 0.68, 0.60, 0.78, 0.70, 0.0])
    cfg = orc.Config(cells=(L, L, L), model=0, T=700.0, seed=91)
    nn = np.array([[_is_1nn(a, b, L) for b in range(n)] for a in range(n)])
    idx = -np.ones((n, n), dtype=np.int64)          # state (v, c) -> unknown index (non-absorbing only)
    states = [(v, c) for v in range(n) for c in range(n) if v != c and not nn[v, c]]
    for i, (v, c) in enumerate(states):
        idx[v, c] = i
    offs = synth.window_offsets_np()[:8, :3]        # 1NN half-cell offsets, hop order k = 0..7
    rows, cols, vals = [], [], []
    gtot = np.empty(len(states))
    rate_cache = {}
    for i, (v, c) in enumerate(states):
        sp = np.zeros(n, dtype=np.uint8); sp[v] = 6; sp[c] = 1
        _, G, _ = orc.barriers(cfg, sp, v, eps, E0)
        gtot[i] = G.sum()
        rows.append(i); cols.append(i); vals.append(-G.sum())
        pv = _half_cell_pos(np.array([v]), L)[0]
        for k in range(8):
            pn = (pv + offs[k]) % (2 * L)
            t = int(2 * ((pn[0] // 2) + L * ((pn[1] // 2) + L * (pn[2] // 2))) + pn[0] % 2)
            j = idx[t, c]                           # the vacancy moves to t (t != c: c is not a 1NN of v)
            if j >= 0:
                rows.append(i); cols.append(j); vals.append(G[k])
        rate_cache[(v, c)] = G
    A = csr_matrix((vals, (rows, cols)), shape=(len(states), len(states)))
    tau = spsolve(A.tocsc(), -np.ones(len(states)))
    assert np.all(tau > 0)
    # Monte Carlo: absorption times of serial BKL episodes from one start state
    v0, c0 = 0, 2 * (2 + L * (2 + L * 2))           # Cu two cells away along the body diagonal
    assert idx[v0, c0] >= 0
    times = []
    for ep in range(1500):
        sp = np.zeros(n, dtype=np.uint8); sp[v0] = 6; sp[c0] = 1
        c = orc.Config(cells=(L, L, L), model=0, T=700.0, seed=1000 + ep)
        st = orc.State.from_species(c, sp)
        while not nn[st.vac[0], c0]:
            orc.run(c, st, 1, eps, E0)
        times.append(st.clock[0])
    times = np.array(times)
    t_exact = tau[idx[v0, c0]]
    se = times.std(ddof=1) / math.sqrt(times.size)
    print("mfpt", times.mean(), t_exact, se)
    assert abs(times.mean() - t_exact) < 4 * se, (times.mean(), t_exact, se)
    # Eq. 7 with the exact u = Gamma_tot tau reproduces delta-tau = tau(s) - tau(s') (absorbing: tau = 0)
    u = gtot * tau
    i0 = idx[v0, c0]
    for k in range(8):
        pv = _half_cell_pos(np.array([v0]), L)[0]
        pn = (pv + offs[k]) % (2 * L)
        t = int(2 * ((pn[0] // 2) + L * ((pn[1] // 2) + L * (pn[2] // 2))) + pn[0] % 2)
        j = idx[t, c0]
        tau_n, u_n, g_n = (tau[j], u[j], gtot[j]) if j >= 0 else (0.0, 0.0, 1.0)
        dt_hat = (u[i0] - gtot[i0] / g_n * u_n) / gtot[i0]
        assert dt_hat == pytest.approx(tau[i0] - tau_n, rel=1e-12, abs=1e-30)


def test_anisotropic_hops_are_first_neighbours(orc):
    """Geometry pin on a non-cubic box (each Lx, Ly, Lz even and >= 4, not necessarily equal):
    every event the oracle applies moves one vacancy by a bcc first-neighbour vector (+-1/2, +-1/2, +-1/2)
    cells under the periodic metric of EACH axis (hops go to the 8 first neighbours), composition is
    conserved, and all 8 directions occur.  Brute force from site coordinates, so a transposed axis or a
    stride of the wrong length in the oracle's neighbour table fails here."""
    cells = (6, 10, 14)
    Lx, Ly, Lz = cells
    sp = synth.make_lattice(cells, 1, synth.fe_cu_fractions(0.1), 3, seed=17)
    cfg = orc.Config(cells=cells, model=0, seed=31)
    eps, E0 = synth.illustrative_pair_params()
    st = orc.State.from_species(cfg, sp)
    counts0 = np.bincount(sp, minlength=7)

    def pos2(i):                       # doubled coordinates: 2*cell + basis
        b, c = i % 2, i // 2
        return np.array([2 * (c % Lx) + b, 2 * ((c // Lx) % Ly) + b, 2 * (c // (Lx * Ly)) + b])

    seen = set()
    for _ in range(600):
        before = st.vac.copy()
        assert orc.run(cfg, st, 1, eps, E0) == orc.ORC_OK
        moved = np.flatnonzero(st.vac != before)
        assert moved.size == 1
        d = pos2(st.vac[moved[0]]) - pos2(before[moved[0]])
        d = (d + np.array([Lx, Ly, Lz])) % (2 * np.array([Lx, Ly, Lz])) - np.array([Lx, Ly, Lz])
        assert np.array_equal(np.abs(d), [1, 1, 1]), d
        seen.add(tuple(d))
    assert len(seen) == 8
    assert np.array_equal(np.bincount(st.species, minlength=7), counts0)
    assert np.array_equal(np.sort(st.vac), np.flatnonzero(st.species == 6))
