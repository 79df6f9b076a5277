"""Pins of the oracle's multi-vacancy residence-time selection, -m "not gpu".

Eq. 2 read with log-rate logits is the BKL law: in a competing set of several vacancies
event a = (vacancy i, hop k) is chosen with probability Gamma_a / Gamma_tot, Gamma_tot = sum over ALL
vacancies and hops, and dt * Gamma_tot ~ Exp(1).  The oracle realises the
across-vacancy half with a canonical pairwise tree (tree_build) and a descent (tree_descend), reading
A17.  These tests pin that half with more than one leaf -- 3 and 5 vacancies (not powers of two, so
the tree is padded), unequal R_i, a zero-rate leaf -- against:
  * the exact law, deterministically: stratified u_sel = (j + 1/2)/N hits event a exactly
    N * Gamma_a / Gamma_tot times up to boundary rounding (+-1);
  * Gamma_tot against math.fsum of all rates (the tree is a reordering of an exact-ish sum);
  * S:202's worked example literally (rates 3 Gamma and Gamma -> 0.75 / 0.25 within 3 sigma, 1e5 draws);
  * end to end through orc_run: chi^2 of (vacancy, hop) frequencies over 1e5 seeds and a KS test of
    dt * Gamma_tot against Exp(1), with Gamma_tot = fsum of orc.rates;
and each test is shown to REJECT fault-injected builds of the same oracle (-DORC_MUTANT=k: right turn
without subtracting the left mass, swapped child offsets, a padded tree that drops a real leaf).
"""
import math

import numpy as np
import pytest

import synth

MUTANTS = (1, 2, 3)


def _rates_3_5():
    """Hop-rate tables with unequal R_i: 3 and 5 vacancies, masked hops, one all-zero vacancy."""
    rng = np.random.default_rng(20260419)
    out = {}
    for n in (3, 5):
        G = rng.uniform(0.2, 3.0, size=(n, 8)) * 10.0 ** rng.integers(-1, 2, size=(n, 1))
        G[rng.random((n, 8)) < 0.25] = 0.0          # masked hops (Gamma = 0 exactly)
        if n == 5:
            G[2, :] = 0.0                             # a vacancy with no feasible hop (R_i = 0 leaf)
        out[n] = G
    return out


def _stratified_counts(orc, G, N, L=None):
    counts = np.zeros_like(G, dtype=np.int64)
    tot = None
    for j in range(N):
        t, i, k = orc.bkl_select_u(G, (j + 0.5) / N, L)
        tot = t
        counts[i, k] += 1
    return tot, counts


@pytest.mark.parametrize("n", [3, 5])
def test_stratified_selection_is_exact_law(orc, n):
    """Deterministic: with u_sel on a uniform grid every event is chosen N * Gamma_a / Gamma_tot times
    (+-1 at the cell boundaries); Gamma_tot equals the exact sum to a few ulp."""
    G = _rates_3_5()[n]
    N = 100_000
    tot, counts = _stratified_counts(orc, G, N)
    exact = math.fsum(G.ravel())
    assert abs(tot - exact) <= 4 * math.ulp(exact)
    expected = N * G / exact
    assert np.all(np.abs(counts - expected) <= 1.0 + 1e-9), np.abs(counts - expected).max()
    assert counts[G == 0.0].sum() == 0                 # masked hops / dead vacancy never chosen


def test_stratified_law_rejects_mutants(orc):
    """A wrong descent (no subtraction, swapped children, dropped padded leaf) fails the exact law."""
    G = _rates_3_5()[5]
    N = 20_000
    exact = math.fsum(G.ravel())
    for m in MUTANTS:
        Lm = orc.load_variant(orc.build(mutant=m))
        tot, counts = _stratified_counts(orc, G, N, Lm)
        err = np.abs(counts - N * G / exact).max()
        assert err > 50 or abs(tot - exact) > 1e-6 * exact, f"mutant {m} not detected (err {err})"


def test_spec_three_to_one_example(orc):
    """S:202 literally: two events with rates 3 Gamma and Gamma (two vacancies, one feasible hop each)
    -> frequencies 0.75 / 0.25 within 3 sigma over 1e5 draws of the serial Philox stream."""
    gam = 1.7e6
    G = np.zeros((2, 8))
    G[0, 3] = 3 * gam
    G[1, 6] = gam
    n = 100_000
    first = 0
    for e in range(n):
        u_sel, _ = orc.draw_uniforms(99, (e, 0, 0, 0))    # serial counter (event, 0, voxel 0, 0), A16
        t, i, k = orc.bkl_select_u(G, u_sel)
        assert (i, k) in ((0, 3), (1, 6))
        first += i == 0
    sigma = math.sqrt(n * 0.75 * 0.25)
    assert abs(first - 0.75 * n) < 3 * sigma


def _five_vacancy_lattice(orc, n_vac):
    """8^3-cell Fe voxel, n_vac vacancies 4 cells apart, solute shells around each so R_i differ."""
    L = 8
    sp = np.zeros(2 * L ** 3, dtype=np.uint8)
    w = orc.window_offsets()
    rng = np.random.default_rng(7 + n_vac)
    cells = [(0, 0, 0), (4, 0, 0), (0, 4, 0), (4, 4, 4), (0, 0, 4)][:n_vac]
    sites = []
    for ci, (cx, cy, cz) in enumerate(cells):
        v = 2 * (cx + L * (cy + L * cz))
        sites.append(v)
        # a different solute mix in the first two shells of each vacancy
        for j in range(14):
            if rng.random() < 0.2 + 0.1 * ci:
                p = (np.array([2 * cx + w[j, 0], 2 * cy + w[j, 1], 2 * cz + w[j, 2]])) % (2 * L)
                sp[2 * ((p[0] >> 1) + L * ((p[1] >> 1) + L * (p[2] >> 1))) + (p[0] & 1)] = 1 + (ci + j) % 4
    for v in sites:
        sp[v] = 6
    return L, sp


def _first_events(orc, n_vac, n_seeds, L_lib=None):
    Lc, sp = _five_vacancy_lattice(orc, n_vac)
    eps, E0 = synth.illustrative_pair_params()
    cfg = orc.Config(cells=(Lc, Lc, Lc), model=0)
    st0 = orc.State.from_species(cfg, sp)
    G, _ = orc.rates(cfg, st0.species, st0.vac, eps, E0)
    w = orc.window_offsets()
    # site reached by hop k of each vacancy
    target = np.zeros((n_vac, 8), dtype=np.int64)
    for i, v in enumerate(st0.vac):
        b = v & 1
        c = v >> 1
        x, y, z = c % Lc, (c // Lc) % Lc, c // (Lc * Lc)
        for k in range(8):
            p = (np.array([2 * x + b + w[k, 0], 2 * y + b + w[k, 1], 2 * z + b + w[k, 2]])) % (2 * Lc)
            target[i, k] = 2 * ((p[0] >> 1) + Lc * ((p[1] >> 1) + Lc * (p[2] >> 1))) + (p[0] & 1)
    counts = np.zeros((n_vac, 8), dtype=np.int64)
    dts = np.zeros(n_seeds)
    for s in range(n_seeds):
        cfg.seed = s
        st = st0.copy()
        orc.run(cfg, st, 1, eps, E0, L=L_lib)
        moved = np.flatnonzero(st.vac != st0.vac)
        assert moved.size == 1
        i = int(moved[0])
        k = int(np.flatnonzero(target[i] == st.vac[i])[0])
        counts[i, k] += 1
        dts[s] = st.clock[0]
    return G, counts, dts


@pytest.mark.parametrize("n_vac,n_seeds", [(3, 40_000), (5, 100_000)])
def test_multi_vacancy_selection_end_to_end(orc, n_vac, n_seeds):
    """orc_run over many seeds: chi^2 of the (vacancy, hop) frequencies against Gamma_a / Gamma_tot from
    orc.rates, and dt * Gamma_tot ~ Exp(1) (KS + mean within 4 sigma) with Gamma_tot = fsum(rates)."""
    from scipy import stats
    G, counts, dts = _first_events(orc, n_vac, n_seeds)
    R = G.sum(axis=1)
    assert len(set(np.round(R / R.max(), 6))) == n_vac, R     # unequal R_i (the tree is exercised)
    gtot = math.fsum(G.ravel())
    p = G.ravel() / gtot
    live = p > 0
    assert counts.ravel()[~live].sum() == 0
    assert stats.chisquare(counts.ravel()[live], p[live] * n_seeds).pvalue > 1e-3
    x = dts * gtot
    assert stats.kstest(x, "expon").pvalue > 1e-3
    assert abs(x.mean() - 1.0) < 4.0 / math.sqrt(n_seeds)


def test_end_to_end_rejects_mutants(orc):
    """The same chi^2 / Exp(1) pair fails for every fault-injected descent (5 vacancies, 2e4 seeds)."""
    from scipy import stats
    for m in MUTANTS:
        Lm = orc.load_variant(orc.build(mutant=m))
        G, counts, dts = _first_events(orc, 5, 20_000, L_lib=Lm)
        gtot = math.fsum(G.ravel())
        p = G.ravel() / gtot
        live = p > 0
        dead_hits = counts.ravel()[~live].sum()
        chi_p = stats.chisquare(counts.ravel()[live], p[live] * counts.sum()).pvalue if dead_hits == 0 else 0.0
        ks_p = stats.kstest(dts * gtot, "expon").pvalue
        assert min(chi_p, ks_p) < 1e-6, f"mutant {m} not detected (chi2 p {chi_p:.3g}, KS p {ks_p:.3g})"
