"""ctypes wrapper of the plain-C FP64 oracle (oracle/akmc_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_2604_24091_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "akmc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ORC_OK, ORC_INVALID, ORC_TERMINAL = 0, 2, 3


def build(force: bool = False, mutant: int = 0) -> str:
    """Compile the oracle: plain C11, -O2, no SIMD intrinsics, no FP contraction.  mutant != 0 builds a
    separate fault-injected copy (liboracle_mutant<k>.so, -DORC_MUTANT=k) that the selection-law tests
    must reject; the real library is always built with ORC_MUTANT = 0."""
    out = _LIB if not mutant else os.path.join(_HERE, f"liboracle_mutant{int(mutant)}.so")
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               f"-DORC_MUTANT={int(mutant)}", "-o", out + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(out + ".tmp", out)
    return out


class _Cfg(C.Structure):
    _fields_ = [("cells", C.c_int32 * 3), ("n_voxels", C.c_int32), ("T", C.c_double),
                ("nu0", C.c_double), ("kB", C.c_double), ("model", C.c_int32),
                ("domain", C.c_int32 * 3), ("window_s", C.c_double), ("seed", C.c_uint64),
                ("strict", C.c_int32), ("voxel_T", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER
        _lib.orc_philox.argtypes = [P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
        _lib.orc_det_exp.argtypes = [C.c_double]; _lib.orc_det_exp.restype = C.c_double
        _lib.orc_det_log.argtypes = [C.c_double]; _lib.orc_det_log.restype = C.c_double
        _lib.orc_det_exp_n.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
        _lib.orc_det_log_n.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
        _lib.orc_window_offsets.argtypes = [P(C.c_int32)]
        _lib.orc_system_energy.argtypes = [P(_Cfg), C.c_void_p, C.c_int64, C.c_void_p]
        _lib.orc_system_energy.restype = C.c_double
        _lib.orc_delta_energy.argtypes = [P(_Cfg), C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
        _lib.orc_delta_energy.restype = C.c_double
        _lib.orc_window.argtypes = [P(_Cfg), C.c_void_p, C.c_int64, C.c_void_p]
        _lib.orc_mlp_fp64.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_barriers.argtypes = [P(_Cfg), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_run.argtypes = [P(_Cfg), C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        _lib.orc_run_until.argtypes = [P(_Cfg), C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int64, C.c_void_p]
        _lib.orc_rates.argtypes = [P(_Cfg), C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_cluster_stats.argtypes = [P(_Cfg), C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                           C.c_void_p, C.c_void_p, C.c_int64]
        _lib.orc_sector_perm.argtypes = [C.c_uint64, C.c_int64, P(C.c_int)]
        _declare_selection(_lib)
        _lib.orc_softplus.argtypes = [C.c_double]; _lib.orc_softplus.restype = C.c_double
        _lib.orc_delta_tau_hat.argtypes = [C.c_double] * 4; _lib.orc_delta_tau_hat.restype = C.c_double
        _lib.orc_poisson_net.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        _lib.orc_poisson_net.restype = C.c_double
        _lib.orc_run_world.argtypes = [P(_Cfg), C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double,
                                       C.c_int64, C.c_void_p]
        _lib.orc_world_eval.argtypes = [P(_Cfg), C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_void_p,
                                        C.c_void_p, C.c_void_p]
    return _lib


def _declare_selection(L):
    P = C.POINTER
    L.orc_bkl_select_u.argtypes = [C.c_void_p, C.c_int, C.c_double, P(C.c_int), P(C.c_int)]
    L.orc_bkl_select_u.restype = C.c_double
    L.orc_draw_uniforms.argtypes = [C.c_uint64, P(C.c_uint32), P(C.c_double), P(C.c_double)]


def bkl_select_u(G, u_sel: float, L=None):
    """One residence-time selection (the oracle's tree + descent + pick_hop) over hop rates G[n][8] with a
    given u_sel; returns (Gamma_tot, vacancy i, hop k).  L: an alternative build (mutant tests)."""
    g = np.ascontiguousarray(G, dtype=np.float64).reshape(-1, 8)
    i, k = C.c_int(), C.c_int()
    tot = (L or lib()).orc_bkl_select_u(_ptr(g), int(g.shape[0]), float(u_sel), C.byref(i), C.byref(k))
    return tot, i.value, k.value


def draw_uniforms(seed: int, ctr) -> tuple:
    c = (C.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    us, ut = C.c_double(), C.c_double()
    lib().orc_draw_uniforms(int(seed) & 0xFFFFFFFFFFFFFFFF, c, C.byref(us), C.byref(ut))
    return us.value, ut.value


def load_variant(path: str):
    """ctypes handle of an alternative oracle build (fault-injected copies for the selection tests)."""
    L = C.CDLL(path)
    _declare_selection(L)
    P = C.POINTER
    L.orc_run.argtypes = [P(_Cfg), C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    L.orc_rates.argtypes = [P(_Cfg), C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                            C.c_void_p, C.c_void_p, C.c_void_p]
    return L


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class Config:
    cells: tuple = (16, 16, 16)
    n_voxels: int = 1
    T: float = 563.0
    nu0: float = 6.0e12
    kB: float = 8.617333262e-5
    model: int = 0           # 0 pair KRA, 1 MLP
    domain: tuple = (0, 0, 0)
    window_s: float = 0.0
    seed: int = 1
    strict: int = 0
    voxel_T: tuple = None    # per-voxel temperature K (C4 variant) or None = T everywhere

    def c(self) -> _Cfg:
        s = _Cfg()
        s.cells[:] = [int(v) for v in self.cells]
        s.n_voxels = int(self.n_voxels)
        s.T, s.nu0, s.kB = float(self.T), float(self.nu0), float(self.kB)
        s.model = int(self.model)
        s.domain[:] = [int(v) for v in self.domain]
        s.window_s = float(self.window_s)
        s.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        s.strict = int(self.strict)
        if self.voxel_T is not None:
            vt = np.ascontiguousarray(self.voxel_T, dtype=np.float64)
            assert vt.shape == (self.n_voxels,), vt.shape
            s._vt = vt                          # keeps the array alive with the struct
            s.voxel_T = vt.ctypes.data
        return s

    @property
    def sites_per_voxel(self) -> int:
        return 2 * self.cells[0] * self.cells[1] * self.cells[2]


def philox(ctr, key):
    c = (C.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (C.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (C.c_uint32 * 4)()
    lib().orc_philox(c, k, o)
    return list(o)


def det_exp(x: float) -> float:
    return lib().orc_det_exp(float(x))


def det_log(u: float) -> float:
    return lib().orc_det_log(float(u))


def det_exp_n(x) -> np.ndarray:
    xs = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(xs)
    lib().orc_det_exp_n(_ptr(xs), int(xs.size), _ptr(y))
    return y


def det_log_n(x) -> np.ndarray:
    xs = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(xs)
    lib().orc_det_log_n(_ptr(xs), int(xs.size), _ptr(y))
    return y


def window_offsets() -> np.ndarray:
    out = np.zeros((64, 4), dtype=np.int32)
    n = lib().orc_window_offsets(out.ctypes.data_as(C.POINTER(C.c_int32)))
    assert n == 64, n
    return out


def sector_perm(seed: int, sweep: int):
    p = (C.c_int * 8)()
    lib().orc_sector_perm(int(seed) & 0xFFFFFFFFFFFFFFFF, int(sweep), p)
    return list(p)


def system_energy(cfg: Config, species: np.ndarray, vox: int, eps: np.ndarray) -> float:
    sp = np.ascontiguousarray(species, dtype=np.uint8)
    e = np.ascontiguousarray(eps, dtype=np.float64)
    return lib().orc_system_energy(C.byref(cfg.c()), _ptr(sp), int(vox), _ptr(e))


def delta_energy(cfg: Config, species, vsite: int, k: int, eps) -> float:
    sp = np.ascontiguousarray(species, dtype=np.uint8)
    e = np.ascontiguousarray(eps, dtype=np.float64)
    return lib().orc_delta_energy(C.byref(cfg.c()), _ptr(sp), int(vsite), int(k), _ptr(e))


def window(cfg: Config, species, vsite: int) -> np.ndarray:
    sp = np.ascontiguousarray(species, dtype=np.uint8)
    out = np.zeros(64, dtype=np.uint8)
    lib().orc_window(C.byref(cfg.c()), _ptr(sp), int(vsite), _ptr(out))
    return out


def mlp_fp64(sigma: np.ndarray, mlp: np.ndarray) -> np.ndarray:
    s = np.ascontiguousarray(sigma, dtype=np.uint8)
    m = np.ascontiguousarray(mlp, dtype=np.float64)
    E = np.zeros(8)
    lib().orc_mlp_fp64(_ptr(s), _ptr(m), _ptr(E))
    return E


def barriers(cfg: Config, species, vsite: int, eps=None, E0=None, mlp=None):
    sp = np.ascontiguousarray(species, dtype=np.uint8)
    e = None if eps is None else np.ascontiguousarray(eps, dtype=np.float64)
    e0 = None if E0 is None else np.ascontiguousarray(E0, dtype=np.float64)
    m = None if mlp is None else np.ascontiguousarray(mlp, dtype=np.float64)
    E = np.zeros(8); G = np.zeros(8)
    clamps = lib().orc_barriers(C.byref(cfg.c()), _ptr(sp), int(vsite), _ptr(e), _ptr(e0), _ptr(m),
                                _ptr(E), _ptr(G))
    return E, G, clamps


@dataclass
class State:
    species: np.ndarray      # uint8, n_voxels * sites
    vac: np.ndarray          # int64 global site ids, slot order
    clock: np.ndarray        # float64 per voxel
    nev: np.ndarray          # int64 per voxel (serial event counter)
    sweep: np.ndarray        # int64[1]
    counters: np.ndarray     # int64[4] events, hop_evals, terminal_voxels, clamps

    @staticmethod
    def from_species(cfg: Config, species: np.ndarray) -> "State":
        sp = np.ascontiguousarray(species, dtype=np.uint8).copy()
        vac = np.flatnonzero(sp == 6).astype(np.int64)       # slot = rank of initial site
        return State(sp, vac, np.zeros(cfg.n_voxels), np.zeros(cfg.n_voxels, dtype=np.int64),
                     np.zeros(1, dtype=np.int64), np.zeros(4, dtype=np.int64))

    def copy(self) -> "State":
        return State(self.species.copy(), self.vac.copy(), self.clock.copy(), self.nev.copy(),
                     self.sweep.copy(), self.counters.copy())


def run(cfg: Config, st: State, n: int, eps=None, E0=None, mlp=None, L=None) -> int:
    e = None if eps is None else np.ascontiguousarray(eps, dtype=np.float64)
    e0 = None if E0 is None else np.ascontiguousarray(E0, dtype=np.float64)
    m = None if mlp is None else np.ascontiguousarray(mlp, dtype=np.float64)
    return (L or lib()).orc_run(C.byref(cfg.c()), _ptr(st.species), _ptr(st.vac), int(st.vac.size), _ptr(st.clock),
                         _ptr(st.nev), _ptr(st.sweep), _ptr(e), _ptr(e0), _ptr(m), int(n), _ptr(st.counters))


def run_until(cfg: Config, st: State, t_end: float, max_events: int, eps=None, E0=None, mlp=None) -> int:
    """Serial mode: every voxel advances to physical time t_end (<= max_events events each)."""
    e = None if eps is None else np.ascontiguousarray(eps, dtype=np.float64)
    e0 = None if E0 is None else np.ascontiguousarray(E0, dtype=np.float64)
    m = None if mlp is None else np.ascontiguousarray(mlp, dtype=np.float64)
    return lib().orc_run_until(C.byref(cfg.c()), _ptr(st.species), _ptr(st.vac), int(st.vac.size), _ptr(st.clock),
                               _ptr(st.nev), _ptr(e), _ptr(e0), _ptr(m), float(t_end), int(max_events),
                               _ptr(st.counters))


def rates(cfg: Config, species, vac, eps=None, E0=None, mlp=None):
    sp = np.ascontiguousarray(species, dtype=np.uint8)
    v = np.ascontiguousarray(vac, dtype=np.int64)
    e = None if eps is None else np.ascontiguousarray(eps, dtype=np.float64)
    e0 = None if E0 is None else np.ascontiguousarray(E0, dtype=np.float64)
    m = None if mlp is None else np.ascontiguousarray(mlp, dtype=np.float64)
    R = np.zeros((v.size, 8)); E = np.zeros((v.size, 8))
    lib().orc_rates(C.byref(cfg.c()), _ptr(sp), _ptr(v), int(v.size), _ptr(e), _ptr(e0), _ptr(m), _ptr(R), _ptr(E))
    return R, E


def cluster_stats(cfg: Config, species, vox: int = 0, cu: int = 1, nstar: int = 4, hist_len: int = 64):
    sp = np.ascontiguousarray(species, dtype=np.uint8)
    out = np.zeros(8); hist = np.zeros(hist_len, dtype=np.int64)
    lib().orc_cluster_stats(C.byref(cfg.c()), _ptr(sp), int(vox), int(cu), int(nstar), _ptr(out), _ptr(hist),
                            int(hist_len))
    keys = ["n_cu", "n_clusters", "n_clusters2", "largest", "monomers", "precipitates", "mean_size2",
            "cucu_bonds"]
    d = {k: float(v) for k, v in zip(keys, out)}
    d["hist"] = hist
    return d


# ----------------------------------------------------------------------------- world-model time mode (f2)
def softplus(y: float) -> float:
    return lib().orc_softplus(float(y))


def delta_tau_hat(u_s: float, g_s: float, u_sp: float, g_sp: float) -> float:
    """Eq. 7: (u(s) - Gamma_tot(s)/Gamma_tot(s') u(s')) / Gamma_tot(s)."""
    return lib().orc_delta_tau_hat(float(u_s), float(g_s), float(u_sp), float(g_sp))


def poisson_net(sigmas, tnet, H: int) -> float:
    s = np.ascontiguousarray(sigmas, dtype=np.uint8).reshape(-1, 64)
    t = np.ascontiguousarray(tnet, dtype=np.float64)
    return lib().orc_poisson_net(_ptr(s), int(s.shape[0]), _ptr(t), int(H))


def run_world(cfg: Config, st: State, n: int, eps, E0, mlp, tnet, H: int, tau_act: float = 1.0) -> int:
    """Serial world-model steps (policy-logit selection, Eq. 7 clock), n events per voxel."""
    e = np.ascontiguousarray(eps, dtype=np.float64)
    e0 = np.ascontiguousarray(E0, dtype=np.float64)
    m = np.ascontiguousarray(mlp, dtype=np.float64)
    t = np.ascontiguousarray(tnet, dtype=np.float64)
    return lib().orc_run_world(C.byref(cfg.c()), _ptr(st.species), _ptr(st.vac), int(st.vac.size), _ptr(st.clock),
                               _ptr(st.nev), _ptr(e), _ptr(e0), _ptr(m), _ptr(t), int(H), float(tau_act), int(n),
                               _ptr(st.counters))


def world_eval(cfg: Config, species, vac, vox: int, eps, E0, mlp, tnet, H: int, tau_act: float = 1.0):
    """(policy weights W[m][8], physical rates G[m][8], wtot, gtot, uhat) of voxel `vox`."""
    sp = np.ascontiguousarray(species, dtype=np.uint8)
    v = np.ascontiguousarray(vac, dtype=np.int64)
    W = np.zeros((v.size + 1, 8)); G = np.zeros((v.size + 1, 8)); o = np.zeros(3)
    m = lib().orc_world_eval(C.byref(cfg.c()), _ptr(sp), _ptr(v), int(v.size), int(vox),
                             _ptr(np.ascontiguousarray(eps, dtype=np.float64)),
                             _ptr(np.ascontiguousarray(E0, dtype=np.float64)),
                             _ptr(np.ascontiguousarray(mlp, dtype=np.float64)),
                             _ptr(np.ascontiguousarray(tnet, dtype=np.float64)), int(H), float(tau_act),
                             _ptr(W), _ptr(G), _ptr(o))
    return W[:m], G[:m], o[0], o[1], o[2]
