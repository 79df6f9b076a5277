"""Pins of the oracle's world-model time mode, -m "not gpu".

What the paper fixes (Eqs. 1-2, Eqs. 5-7):
  * Eq. 1/2: masked hops have probability exactly 0; the softmax over the concatenated logits equals the
    factorised Eq. 4 computation; tau_act -> large gives the uniform law over feasible hops;
    with logits z = -E/kT the law is the BKL law Gamma_a / Gamma_tot (the reading that links the two);
  * the selection realised by the oracle (tree + descent over det_exp(zhat)) follows that law (chi^2);
  * Eq. 7 with the exact u = Gamma_tot tau from an MFPT solve (Eq. 5) reproduces delta-tau = tau(s) - tau(s')
    (plug-in identity S:399), telescopes to tau(s0) over a path to absorption, and equals
    c (1 - Gamma(s)/Gamma(s')) / Gamma(s) for a constant uhat = c;
  * softplus (the Poisson net's head) against libm; the pooled Poisson net against a closed form;
  * one world step's clock increment = max(Eq. 7, 1e-3 / Gamma_tot(s)) recomputed from world_eval.
"""
import math

import numpy as np
import pytest

import synth
from mfpt_space import mfpt_space as _mfpt_space

KT = 8.617333262e-5 * 563.0


def _lattice(L=8, n_vac=3, seed=5):
    return synth.make_lattice((L, L, L), 1, synth.fe_cu_fractions(0.05), n_vac, seed=seed)


def _nets(seed=1, H=16):
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.random_mlp(seed=seed)
    return eps, E0, mlp, synth.poisson_net(seed + 10, H=H), H


def test_softplus_against_libm(orc):
    for y in [-40.0, -5.0, -0.3, 0.0, 1e-8, 0.7, 3.0, 25.0, 80.0]:
        ref = math.log1p(math.exp(y)) if y < 30 else y + math.log1p(math.exp(-y))
        got = orc.softplus(y)
        assert got >= 0.0
        # ln(1 + x) as det_log(1 + x): the rounding of 1 + x bounds the ABSOLUTE error by ~ulp(1)
        assert got == pytest.approx(ref, rel=4e-15, abs=4e-16), (y, got, ref)
    assert orc.softplus(0.0) == pytest.approx(math.log(2.0), rel=1e-15)


def test_poisson_net_closed_form_and_pooling(orc):
    """H = 1, Wt1 = one-hot of feature f0, bt1 = 0, wt2 = 1, bt2 = b: uhat = softplus(count_f0 / n + b); the
    pooled input is a mean, so the vacancy order does not matter (bit-identical)."""
    rng = np.random.default_rng(3)
    wins = synth.random_windows(5, seed=4)
    for f0 in (0, 7 * 3 + 2, 7 * 63 + 6):
        H = 1
        t = np.zeros(448 * H + 2 * H + 1)
        t[f0] = 1.0
        t[448 + 1] = 1.0
        t[-1] = -0.25
        cnt = sum(int(w[f0 // 7] == f0 % 7) for w in wins)
        assert orc.poisson_net(wins, t, H) == pytest.approx(math.log1p(math.exp(cnt / 5 - 0.25)), rel=1e-14)
    t = synth.poisson_net(9, H=24)
    a = orc.poisson_net(wins, t, 24)
    b = orc.poisson_net(wins[rng.permutation(5)], t, 24)
    assert a == b and a > 0.0


def test_eq2_masks_softmax_and_factorisation(orc):
    """Policy weights of a voxel: masked hops weight exactly 0; W / sum W == softmax of the concatenated
    logits (Eq. 2) == the factorised Eq. 4 over distinct contexts (to 1e-12)."""
    eps, E0, mlp, tnet, H = _nets()
    L = 8
    sp = _lattice(L, 4, seed=8)
    vac = np.flatnonzero(sp == 6)
    cfg = orc.Config(cells=(L, L, L), model=1)
    W, G, wtot, gtot, uhat = orc.world_eval(cfg, sp, vac, 0, eps, E0, mlp, tnet, H)
    # independent logits: numpy forward pass of the one-hot windows (library matmuls, no clamp)
    W1, b1, W2, b2, W3, b3 = synth.split_mlp(mlp)
    wins = np.stack([orc.window(cfg, sp, int(v)) for v in vac])
    X = np.zeros((len(vac), 448))
    X[np.arange(len(vac))[:, None], 7 * np.arange(64)[None, :] + wins] = 1.0
    z_np = np.maximum(np.maximum(X @ W1 + b1, 0) @ W2 + b2, 0) @ W3 + b3
    M = wins[:, :8] != 6
    assert np.all(W[~M] == 0.0)
    z = np.where(M, z_np, -np.inf)
    p_softmax = np.exp(z - z[M].max()) / np.exp(z - z[M].max()).sum()
    assert np.allclose(W / W.sum(), p_softmax, rtol=1e-12, atol=0)
    # Eq. 4: contexts = distinct windows; nu(u) = multiplicity; per-agent probability = Pr(u,k) / nu(u)
    keys = [orc.window(cfg, sp, int(v)).tobytes() for v in vac]
    nu = {k: keys.count(k) for k in keys}
    den = sum(nu[k] * np.exp(z[i][M[i]]).sum() for i, k in enumerate(keys) if i == keys.index(k))
    for i, k in enumerate(keys):
        pr = nu[k] * np.exp(z[i]) / den
        assert np.allclose(pr / nu[k], W[i] / W.sum(), rtol=1e-12, atol=1e-300)
    assert wtot == pytest.approx(math.fsum(W.ravel()), rel=1e-15)
    assert gtot == pytest.approx(math.fsum(G.ravel()), rel=1e-15)


def test_policy_from_barriers_is_bkl_law(orc):
    """Reading W2: logits z = -E/kT (synth.policy_mlp of the physics network) make Eq. 2's law the BKL law:
    W / sum W == Gamma / sum Gamma of the same network's barriers."""
    eps, E0 = synth.illustrative_pair_params()
    phys = synth.physics_mlp(eps, E0)
    pol = synth.policy_mlp(phys, KT)
    tnet, H = synth.poisson_net(2, H=8), 8
    L = 8
    sp = _lattice(L, 3, seed=11)
    vac = np.flatnonzero(sp == 6)
    cfg = orc.Config(cells=(L, L, L), model=1)
    W, _, _, _, _ = orc.world_eval(cfg, sp, vac, 0, eps, E0, pol, tnet, H)
    Gb, _ = orc.rates(cfg, sp, vac, mlp=phys)
    assert np.allclose(W / W.sum(), Gb / Gb.sum(), rtol=1e-12, atol=1e-300)


def test_tau_act_limit_is_uniform(orc):
    """tau_act -> large: the softmax over unmasked entries is uniform within 1e-6 at tau_act = 1e6."""
    eps, E0, mlp, tnet, H = _nets()
    L = 8
    sp = _lattice(L, 3, seed=13)
    vac = np.flatnonzero(sp == 6)
    cfg = orc.Config(cells=(L, L, L), model=1)
    W, _, _, _, _ = orc.world_eval(cfg, sp, vac, 0, eps, E0, mlp, tnet, H, tau_act=1e6)
    p = W / W.sum()
    live = W > 0
    assert np.allclose(p[live], 1.0 / live.sum(), rtol=1e-6)


def test_world_selection_law_chi2(orc):
    """The oracle's world step selects (vacancy, hop) with probability W / sum W (chi^2 over 2e4 seeds)."""
    from scipy import stats
    eps, E0, mlp, tnet, H = _nets(seed=3)
    L = 8
    sp = _lattice(L, 3, seed=17)
    cfg = orc.Config(cells=(L, L, L), model=1)
    st0 = orc.State.from_species(cfg, sp)
    W, _, _, _, _ = orc.world_eval(cfg, sp, st0.vac, 0, eps, E0, mlp, tnet, H)
    w = orc.window_offsets()
    counts = np.zeros_like(W)
    n = 20000
    for s in range(n):
        cfg.seed = s
        st = st0.copy()
        assert orc.run_world(cfg, st, 1, eps, E0, mlp, tnet, H) == orc.ORC_OK
        i = int(np.flatnonzero(st.vac != st0.vac)[0])
        v = int(st0.vac[i]); b = v & 1; c = v >> 1
        x, y, z = c % L, (c // L) % L, c // (L * L)
        for k in range(8):
            p = (np.array([2 * x + b, 2 * y + b, 2 * z + b]) + w[k, :3]) % (2 * L)
            if 2 * ((p[0] >> 1) + L * ((p[1] >> 1) + L * (p[2] >> 1))) + (p[0] & 1) == st.vac[i]:
                counts[i, k] += 1
    live = W.ravel() > 0
    assert counts.ravel()[~live].sum() == 0
    assert stats.chisquare(counts.ravel()[live], W.ravel()[live] / W.sum() * n).pvalue > 1e-3


def test_world_step_clock_is_eq7(orc):
    """One world step: the clock advances by max(Eq. 7, 1e-3 / Gamma_tot(s)) with uhat and Gamma_tot of the
    states before and after the hop (world_eval), to the bit."""
    eps, E0, mlp, tnet, H = _nets(seed=5)
    L = 8
    sp = _lattice(L, 4, seed=19)
    cfg = orc.Config(cells=(L, L, L), model=1, seed=42)
    st = orc.State.from_species(cfg, sp)
    for _ in range(20):
        _, _, _, g_s, u_s = orc.world_eval(cfg, st.species, st.vac, 0, eps, E0, mlp, tnet, H)
        c0 = st.clock[0]
        orc.run_world(cfg, st, 1, eps, E0, mlp, tnet, H)
        _, _, _, g_sp, u_sp = orc.world_eval(cfg, st.species, st.vac, 0, eps, E0, mlp, tnet, H)
        dt = (u_s - (g_s / g_sp) * u_sp) / g_s
        assert st.clock[0] == c0 + max(dt, 1e-3 / g_s)
        assert orc.delta_tau_hat(u_s, g_s, u_sp, g_sp) == dt


def test_eq7_plugin_identity_and_telescoping(orc):
    tau, gt, succ = _mfpt_space(orc)
    u = gt * tau
    # Eq. 5 residual
    res = [sum(g * ((tau[j] if j >= 0 else 0.0) - tau[i]) for g, j in succ[i]) + 1.0 for i in range(len(tau))]
    assert max(abs(r) for r in res) < 1e-9
    rng = np.random.default_rng(0)
    # plug-in identity on every transition of 300 random states
    for i in rng.choice(len(tau), 300, replace=False):
        for g, j in succ[i]:
            if g == 0.0:
                continue
            if j >= 0:
                got = orc.delta_tau_hat(u[i], gt[i], u[j], gt[j])
                assert got == pytest.approx(tau[i] - tau[j], rel=1e-10, abs=1e-12 * tau[i])
            else:                                       # absorbing s': u(s') = 0 -> tau(s) (S:399 first example)
                assert orc.delta_tau_hat(u[i], gt[i], 0.0, 0.0) == pytest.approx(tau[i], rel=1e-14)
    # telescoping along random paths to absorption: sum of dtau = tau(s0)
    for start in rng.choice(len(tau), 20, replace=False):
        i, total = int(start), 0.0
        for _ in range(100000):
            g, j = succ[i][int(rng.integers(0, 8))]
            if g == 0.0:
                continue
            total += orc.delta_tau_hat(u[i], gt[i], u[j] if j >= 0 else 0.0, gt[j] if j >= 0 else 0.0)
            if j < 0:
                break
            i = j
        assert total == pytest.approx(tau[start], rel=1e-9)
    # constant uhat = c
    c = 0.37
    i = 5
    g, j = next((g, j) for g, j in succ[i] if j >= 0 and g > 0)
    assert orc.delta_tau_hat(c, gt[i], c, gt[j]) == pytest.approx(c * (1 - gt[i] / gt[j]) / gt[i], rel=1e-14)
