"""GPU MFPT solver (akmc_mfpt_solve, Eq. 5): tau on an enumerated state space
against the closed forms SPEC gives (one state -> 1/Gamma; chain A -> B -> absorbing -> 1/G1 + 1/G2)
and against the sparse direct solve of the 16,256-state lattice space whose tau the oracle tests pin to the
BKL dynamics (tests/test_oracle_dynamics.py::test_mfpt_poisson_equation)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def akmc():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_24091_b200 as A
    from paper_2604_24091_b200 import build
    build.build()
    return A


def test_mfpt_closed_forms(akmc):
    tau, it, res = akmc.mfpt_solve([0, 1], [-1], [3.7e5])
    assert tau[0] == pytest.approx(1.0 / 3.7e5, rel=1e-13)
    g1, g2 = 2.0e6, 5.0e4
    tau, it, res = akmc.mfpt_solve([0, 1, 2], [1, -1], [g1, g2])          # A -> B -> absorbing
    assert tau[0] == pytest.approx(1.0 / g1 + 1.0 / g2, rel=1e-12)
    assert tau[1] == pytest.approx(1.0 / g2, rel=1e-12)
    with pytest.raises(akmc.AkmcError):
        akmc.mfpt_solve([0, 0], np.zeros(0, np.int32), np.zeros(0))       # a transient state with no event


def test_mfpt_lattice_space_matches_direct_solve(akmc, orc):
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from mfpt_space import mfpt_space
    tau_ref, gt, succ, (rp, col, rate) = mfpt_space(orc, with_csr=True)
    tau, it, res = akmc.mfpt_solve(rp, col, rate, tol=1e-13)
    assert res < 1e-12, res
    assert np.allclose(tau, tau_ref, rtol=1e-9, atol=0), np.abs(tau / tau_ref - 1).max()
    # Eq. 5 residual with the GPU tau
    r = np.array([sum(g * ((tau[j] if j >= 0 else 0.0) - tau[i]) for g, j in succ[i]) + 1.0 for i in range(len(tau))])
    assert np.abs(r).max() < 1e-8
