"""Time the GPU MFPT solver (akmc_mfpt_solve, Eq. 5) on synthetic enumerated
state spaces shaped like the AKMC ones: every state has 8 events (hops) with Arrhenius rates nu0 exp(-E/kT),
E ~ U(0.4, 0.9) eV at 563 K (rates spanning ~4 decades), targets random states or, with probability p_abs, the
absorbing set.  Beside it: scipy's BiCGSTAB with the same Jacobi preconditioner on the host (one core), and the
residual of Eq. 5 of both answers.

  python tools/mfpt_probe.py [n ...]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def space(n, seed=0, p_abs=0.02):
    rng = np.random.default_rng(seed)
    k = 8
    col = rng.integers(0, n, size=n * k).astype(np.int32)
    col[rng.random(n * k) < p_abs] = -1
    E = rng.uniform(0.4, 0.9, size=n * k)
    rate = 1e13 * np.exp(-E / (8.617333262e-5 * 563.0))
    rp = np.arange(0, n * k + 1, k, dtype=np.int64)
    return rp, col, rate


def residual(rp, col, rate, tau):
    n = rp.size - 1
    row = np.repeat(np.arange(n), np.diff(rp))
    diag = np.bincount(row, weights=rate, minlength=n)
    t = np.where(col >= 0, tau[np.maximum(col, 0)], 0.0)
    off = np.bincount(row, weights=rate * t, minlength=n)
    r = 1.0 - (diag * tau - off)
    return float(np.linalg.norm(r) / np.sqrt(n))


def main():
    import paper_2604_24091_b200 as akmc
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    sizes = [int(a) for a in sys.argv[1:]] or [16384, 131072, 1048576]
    for n in sizes:
        rp, col, rate = space(n)
        akmc.mfpt_solve([0, 1], [-1], [1.0])                                  # (context warm-up)
        t0 = time.perf_counter()
        tau, it, res = akmc.mfpt_solve(rp, col, rate, tol=1e-12)
        t_gpu = time.perf_counter() - t0
        # host: the same Krylov method and preconditioner (scipy, one core)
        row = np.repeat(np.arange(n), 8)
        keep = col >= 0
        A = sp.csr_matrix((-rate[keep], (row[keep], col[keep])), shape=(n, n))
        d = np.bincount(row, weights=rate, minlength=n)
        A = (sp.csr_matrix(A) + sp.diags(d)).tocsr()
        M = sp.diags(1.0 / d)
        t0 = time.perf_counter()
        x, info = spl.bicgstab(A, np.ones(n), rtol=1e-12, atol=0.0, M=M, maxiter=100000)
        t_cpu = time.perf_counter() - t0
        print(json.dumps({"states": n, "nnz": int(rp[-1]), "gpu_s": t_gpu, "iterations": it, "gpu_resid": res,
                          "gpu_resid_recomputed": residual(rp, col, rate, tau), "cpu_bicgstab_s": t_cpu,
                          "cpu_info": int(info), "cpu_resid": residual(rp, col, rate, x),
                          "max_rel_diff_gpu_cpu": float(np.max(np.abs(tau / x - 1.0)))}), flush=True)


if __name__ == "__main__":
    main()
