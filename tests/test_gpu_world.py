"""GPU parity of the world-model time mode (akmc_set_world_model): policy-logit selection
(Eqs. 1-2) and the Eq. 7 clock, FP64, bit-exact against the oracle's orc_run_world -- lattices, vacancy lists,
per-voxel clocks and event counts -- in one voxel (C1 geometry) and a voxel batch with per-voxel T."""
import numpy as np
import pytest

import synth

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


def _run_pair(akmc, orc, cells, nvox, n_vac, seed, n, chunks, mlp, tnet, H, tau=1.0, voxel_T=None):
    eps, E0 = synth.illustrative_pair_params()
    sp = synth.make_lattice(cells, nvox, synth.a508_atomic_fractions(), n_vac, seed=seed)
    cfg = akmc.Config(cells=cells, n_voxels=nvox, barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP64, seed=seed + 1)
    ocfg = orc.Config(cells=cells, n_voxels=nvox, model=1, seed=seed + 1,
                      voxel_T=None if voxel_T is None else tuple(voxel_T))
    st = orc.State.from_species(ocfg, sp)
    with akmc.Simulation(cfg, sp, eps, E0, mlp) as sim:
        if voxel_T is not None:
            sim.set_voxel_temperatures(voxel_T)
        sim.set_world_model(tnet, H, tau)
        ev = 0
        for _ in range(chunks):
            c = sim.step(n // chunks)
            ev += c["events"]
            orc.run_world(ocfg, st, n // chunks, eps, E0, mlp, tnet, H, tau)
        gsp, gvac, gclock, gctr = sim.state()
    return st, (gsp, gvac, gclock, ev)


def test_world_mode_single_voxel_bitexact(akmc, orc):
    """C1 geometry (16^3, Fe-Cu), 2 vacancies, 2000 world steps in 4 calls: bit-exact incl. the Eq. 7 clock."""
    mlp = synth.random_mlp(seed=21)
    tnet = synth.poisson_net(22, H=32)
    st, (gsp, gvac, gclock, ev) = _run_pair(akmc, orc, (16, 16, 16), 1, 2, 2605, 2000, 4, mlp, tnet, 32)
    assert ev == st.counters[0] == 2000
    assert np.array_equal(gsp, st.species) and np.array_equal(gvac, st.vac)
    assert np.array_equal(gclock.view(np.uint64), st.clock.view(np.uint64))
    assert gclock[0] > 0.0


def test_world_mode_voxel_batch_bitexact(akmc, orc):
    """6 voxels of 12^3 with 5 vacancies each, per-voxel T, physics-derived policy (logits -E/kT) and
    tau_act = 0.8: bit-exact per voxel."""
    eps, E0 = synth.illustrative_pair_params()
    pol = synth.policy_mlp(synth.physics_mlp(eps, E0, residual=0.02, seed=3), 8.617333262e-5 * 563.0)
    tnet = synth.poisson_net(5, H=64)
    vT = synth.voxel_temperatures(6, seed=9)
    st, (gsp, gvac, gclock, ev) = _run_pair(akmc, orc, (12, 12, 12), 6, 5, 77, 300, 2, pol, tnet, 64, tau=0.8,
                                            voxel_T=vT)
    assert ev == st.counters[0] == 6 * 300
    assert np.array_equal(gsp, st.species) and np.array_equal(gvac, st.vac)
    assert np.array_equal(gclock.view(np.uint64), st.clock.view(np.uint64))


def test_world_mode_rejects_bad_setups(akmc):
    eps, E0 = synth.illustrative_pair_params()
    mlp = synth.random_mlp(seed=1)
    tnet = synth.poisson_net(2, H=8)
    sp = synth.make_lattice((8, 8, 8), 1, synth.a508_atomic_fractions(), 2, seed=3)
    cfg32 = akmc.Config(cells=(8, 8, 8), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP32)
    with akmc.Simulation(cfg32, sp, eps, E0, mlp) as sim:
        with pytest.raises(akmc.AkmcError):
            sim.set_world_model(tnet, 8)                     # FP64 only
    cfg = akmc.Config(cells=(8, 8, 8), barrier_model=akmc.MODEL_MLP, precision=akmc.PREC_FP64)
    with akmc.Simulation(cfg, sp, None, None, mlp) as sim:
        with pytest.raises(akmc.AkmcError):
            sim.set_world_model(tnet, 8)                     # no eps / E0: no physical rates for Eq. 7
    with akmc.Simulation(cfg, sp, eps, E0, mlp) as sim:
        for bad in [(tnet, 0, 1.0), (tnet, 8, 0.0), (tnet * np.nan, 8, 1.0)]:
            with pytest.raises(akmc.AkmcError):
                sim.set_world_model(*bad)
