"""Enumerable state space of the MFPT tests (test helper, not a test module): L = 4, 1 V + 1 Cu in Fe, absorbing
set = V and Cu first neighbours; rates from the oracle's pair-KRA barriers; tau from a sparse direct solve."""
import numpy as np

import synth


def mfpt_space(orc, with_csr=False):
    """Enumerable space of Eq. 5: L = 4, 1 V + 1 Cu, absorbing = V-Cu first neighbours (as in
    test_oracle_dynamics.test_mfpt_poisson_equation); returns tau, Gamma_tot, successor lists."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.linalg import spsolve
    L = 4
    n = 2 * L ** 3
    eps = np.zeros((2, 7, 7))
    eps[0] = -0.78; eps[1] = -0.39
    eps[0, 6, :] = eps[0, :, 6] = -0.20; eps[0, 6, 1] = eps[0, 1, 6] = -0.33
    E0 = np.array([0.62, 0.54, 0.68, 0.60, 0.78, 0.70, 0.0])
    cfg = orc.Config(cells=(L, L, L), model=0, T=700.0)
    offs = synth.window_offsets_np()[:8, :3]

    def pos(i):
        b = i & 1; c = i >> 1
        return np.array([2 * (c % L) + b, 2 * ((c // L) % L) + b, 2 * (c // (L * L)) + b])

    def site(p):
        p = p % (2 * L)
        return int(2 * ((p[0] // 2) + L * ((p[1] // 2) + L * (p[2] // 2))) + p[0] % 2)

    nn = lambda a, b: any(site(pos(a) + o) == b for o in offs)
    states = [(v, c) for v in range(n) for c in range(n) if v != c and not nn(v, c)]
    idx = {s: i for i, s in enumerate(states)}
    rows, cols, vals, gt, succ = [], [], [], np.empty(len(states)), []
    for i, (v, c) in enumerate(states):
        sp = np.zeros(n, dtype=np.uint8); sp[v] = 6; sp[c] = 1
        _, G, _ = orc.barriers(cfg, sp, v, eps, E0)
        gt[i] = G.sum()
        rows.append(i); cols.append(i); vals.append(-G.sum())
        sl = []
        for k in range(8):
            t = site(pos(v) + offs[k])
            j = idx.get((t, c), -1)
            sl.append((G[k], j))
            if j >= 0:
                rows.append(i); cols.append(j); vals.append(G[k])
        succ.append(sl)
    A = csr_matrix((vals, (rows, cols)), shape=(len(states), len(states)))
    tau = spsolve(A.tocsc(), -np.ones(len(states)))
    if with_csr:
        # transitions per transient state in hop order: (target index or -1 = absorbed, rate)
        rp = np.zeros(len(states) + 1, dtype=np.int64)
        col, rate = [], []
        for i, sl in enumerate(succ):
            for g, j in sl:
                if g > 0.0:
                    col.append(j); rate.append(g)
            rp[i + 1] = len(col)
        return tau, gt, succ, (rp, np.array(col, dtype=np.int32), np.array(rate))
    return tau, gt, succ


