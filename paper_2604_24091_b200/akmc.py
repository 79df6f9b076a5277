"""Thin ctypes binding of include/akmc.h (argument marshalling only; every step of the hot path
runs in the sm_100a kernels of lib/libakmc.so).  There is no CPU fallback: if the library or a
B200 is missing, the calls raise."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# AKMC_LIB: an alternative in-tree build of the same library (A/B timing of kernel variants, tools/ab_probe.py)
LIB_PATH = os.environ.get("AKMC_LIB") or os.path.join(HERE, "lib", "libakmc.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "akmc.h")

AKMC_OK, AKMC_ERR_RUNTIME, AKMC_ERR_INVALID, AKMC_TERMINAL, AKMC_ERR_CUDA, AKMC_ERR_NCCL = range(6)
MODEL_PAIR, MODEL_MLP = 0, 1
PREC_FP64, PREC_FP32, PREC_FP16_FAST = 0, 1, 2
STATUS = {0: "AKMC_OK", 1: "AKMC_ERR_RUNTIME", 2: "AKMC_ERR_INVALID", 3: "AKMC_TERMINAL", 4: "AKMC_ERR_CUDA",
          5: "AKMC_ERR_NCCL"}


class CConfig(C.Structure):
    _fields_ = [("cells", C.c_int32 * 3), ("n_voxels", C.c_int32), ("n_species", C.c_int32),
                ("barrier_model", C.c_int32), ("precision", C.c_int32), ("domain_cells", C.c_int32 * 3),
                ("temperature_K", C.c_double), ("nu0", C.c_double), ("kB", C.c_double), ("window_s", C.c_double),
                ("seed", C.c_uint64), ("gpu_grid", C.c_int32 * 3), ("rank", C.c_int32), ("world", C.c_int32),
                ("nccl_id", C.c_uint8 * 128)]


class CCounters(C.Structure):
    _fields_ = [("events", C.c_int64), ("hop_evals", C.c_int64), ("iterations", C.c_int64), ("clamps", C.c_int64),
                ("terminal_voxels", C.c_int64), ("sweeps", C.c_int64), ("kernel_launches", C.c_int64),
                ("mlp_launches", C.c_int64), ("mlp_rows", C.c_int64), ("mlp_ms", C.c_double), ("wall_ms", C.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class AkmcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


_lib = None


def load() -> C.CDLL:
    """Load lib/libakmc.so (built by paper_2604_24091_b200.build); raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(f"{LIB_PATH} missing: run `python -m paper_2604_24091_b200.build` "
                                "(the AKMC path has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    lib.akmc_init.argtypes = [C.POINTER(CConfig), P, P, P, P, C.POINTER(P)]
    lib.akmc_step.argtypes = [P, C.c_int64, C.POINTER(CCounters)]
    lib.akmc_run_until.argtypes = [P, C.c_double, C.c_int64, C.POINTER(CCounters)]
    lib.akmc_debug_math.argtypes = [C.c_int32, P, C.c_int64, P]
    lib.akmc_state.argtypes = [P, P, P, C.POINTER(C.c_int64), P, C.POINTER(CCounters)]
    lib.akmc_rates.argtypes = [P, P, P]
    lib.akmc_eval_windows.argtypes = [P, P, C.c_int64, C.c_int32, P]
    lib.akmc_vacancies.argtypes = [P, P, P, C.POINTER(C.c_int64)]
    lib.akmc_nccl_unique_id.argtypes = [P]
    lib.akmc_debug_extended.argtypes = [P, P]
    lib.akmc_set_stream.argtypes = [P, P]
    lib.akmc_set_profiling.argtypes = [P, C.c_int32]
    lib.akmc_set_voxel_temperatures.argtypes = [P, P, C.c_int32]
    lib.akmc_progress.argtypes = [P, P, P]
    lib.akmc_set_world_model.argtypes = [P, P, C.c_int32, C.c_double]
    lib.akmc_voxel_order.argtypes = [P, P]
    lib.akmc_exchange_stats.argtypes = [P, P]
    lib.akmc_set_dataflow.argtypes = [P, C.c_int32]
    lib.akmc_mfpt_solve.argtypes = [P, P, P, C.c_int64, C.c_double, C.c_int32, P, C.POINTER(C.c_int32),
                                    C.POINTER(C.c_double)]
    lib.akmc_restore.argtypes = [P, P, C.c_int64, P, P, C.c_int64]
    lib.akmc_free.argtypes = [P]
    lib.akmc_free.restype = None
    lib.akmc_last_error.argtypes = [P]
    lib.akmc_last_error.restype = C.c_char_p
    lib.akmc_version.restype = C.c_char_p
    for n in ("akmc_init", "akmc_step", "akmc_state", "akmc_rates", "akmc_eval_windows", "akmc_set_stream",
              "akmc_set_profiling", "akmc_vacancies", "akmc_nccl_unique_id", "akmc_debug_extended",
              "akmc_set_voxel_temperatures", "akmc_run_until", "akmc_debug_math", "akmc_progress", "akmc_restore",
              "akmc_set_world_model", "akmc_mfpt_solve", "akmc_voxel_order",
              "akmc_exchange_stats", "akmc_set_dataflow"):
        getattr(lib, n).restype = C.c_int
    _lib = lib
    return lib


def header_symbols() -> list:
    """Function names declared in include/akmc.h."""
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(akmc_\w+)\s*\(", txt, re.M)))


@dataclass
class Config:
    cells: tuple = (16, 16, 16)
    n_voxels: int = 1
    barrier_model: int = MODEL_PAIR
    precision: int = PREC_FP64
    domain_cells: tuple = (0, 0, 0)
    temperature_K: float = 563.0
    nu0: float = 6.0e12
    kB: float = 8.617333262e-5
    window_s: float = 0.0
    seed: int = 1
    gpu_grid: tuple = (1, 1, 1)
    rank: int = 0
    world: int = 1
    nccl_id: bytes = b""

    def c(self) -> CConfig:
        s = CConfig()
        s.cells[:] = [int(v) for v in self.cells]
        s.n_voxels = int(self.n_voxels)
        s.n_species = 7
        s.barrier_model = int(self.barrier_model)
        s.precision = int(self.precision)
        s.domain_cells[:] = [int(v) for v in self.domain_cells]
        s.temperature_K, s.nu0, s.kB, s.window_s = (float(self.temperature_K), float(self.nu0), float(self.kB),
                                                    float(self.window_s))
        s.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        s.gpu_grid[:] = [int(v) for v in self.gpu_grid]
        s.rank, s.world = int(self.rank), int(self.world)
        if self.nccl_id:
            s.nccl_id[:] = list(bytes(self.nccl_id)[:128].ljust(128, b"\0"))
        return s

    @property
    def sites(self) -> int:
        return 2 * self.cells[0] * self.cells[1] * self.cells[2] * self.n_voxels


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def debug_math(fn: int, x) -> np.ndarray:
    """The device's det_exp (fn 0) / det_log (fn 1) on host doubles (diagnostics)."""
    lib = load()
    xs = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    y = np.empty_like(xs)
    rc = lib.akmc_debug_math(int(fn), _ptr(xs), int(xs.size), _ptr(y))
    if rc != AKMC_OK:
        raise AkmcError(rc, "akmc_debug_math failed")
    return y


class Simulation:
    """One akmc_handle.  species: uint8 host array (canonical order); eps [2,7,7], E0 [7], mlp flat."""

    def __init__(self, cfg: Config, species, eps=None, E0=None, mlp=None):
        self.lib = load()
        self.cfg = cfg
        sp = np.ascontiguousarray(species, dtype=np.uint8)
        self._eps = None if eps is None else np.ascontiguousarray(eps, dtype=np.float64)
        self._E0 = None if E0 is None else np.ascontiguousarray(E0, dtype=np.float64)
        self._mlp = None if mlp is None else np.ascontiguousarray(mlp, dtype=np.float64)
        h = C.c_void_p()
        cc = cfg.c()
        rc = self.lib.akmc_init(C.byref(cc), _ptr(sp), _ptr(self._eps), _ptr(self._E0), _ptr(self._mlp), C.byref(h))
        if rc != AKMC_OK:
            raise AkmcError(rc, self.lib.akmc_last_error(None).decode())
        self.h = h
        n = C.c_int64(0)
        self._check(self.lib.akmc_state(self.h, None, None, C.byref(n), None, None))
        self.n_vac = int(n.value)

    def _check(self, rc: int, allow=(AKMC_OK,)):
        if rc not in allow:
            raise AkmcError(rc, self.lib.akmc_last_error(self.h).decode())
        return rc

    def step(self, n: int) -> dict:
        ctr = CCounters()
        rc = self._check(self.lib.akmc_step(self.h, int(n), C.byref(ctr)), allow=(AKMC_OK, AKMC_TERMINAL))
        d = ctr.as_dict()
        d["status"] = rc
        return d

    def run_until(self, t_end: float, max_events: int = 1 << 30) -> dict:
        """Voxel-ensemble mode: every voxel advances to physical time t_end (serial mode)."""
        ctr = CCounters()
        rc = self._check(self.lib.akmc_run_until(self.h, float(t_end), int(max_events), C.byref(ctr)),
                         allow=(AKMC_OK, AKMC_TERMINAL))
        d = ctr.as_dict()
        d["status"] = rc
        return d

    def state(self, species=True):
        sp = np.empty(self.cfg.sites, dtype=np.uint8) if species else None
        nv = C.c_int64(0)
        self._check(self.lib.akmc_vacancies(self.h, None, None, C.byref(nv)))
        vac = np.empty(max(int(nv.value), 1), dtype=np.int64)
        n = C.c_int64(vac.size)
        clock = np.empty(self.cfg.n_voxels, dtype=np.float64)
        ctr = CCounters()
        self._check(self.lib.akmc_state(self.h, _ptr(sp), _ptr(vac), C.byref(n), _ptr(clock), C.byref(ctr)))
        return sp, vac[: n.value], clock, ctr.as_dict()

    def counters(self) -> dict:
        """Cumulative counters only (one small device->host read, no lattice or vacancy transfer)."""
        ctr = CCounters()
        self._check(self.lib.akmc_state(self.h, None, None, None, None, C.byref(ctr)))
        return ctr.as_dict()

    def vacancies(self):
        """(global slot ids, global canonical sites) of the vacancies this rank owns, sorted by id."""
        n = C.c_int64(0)
        self._check(self.lib.akmc_vacancies(self.h, None, None, C.byref(n)))
        cap = max(int(n.value), 1)
        gid = np.empty(cap, dtype=np.int64); site = np.empty(cap, dtype=np.int64)
        n = C.c_int64(cap)
        self._check(self.lib.akmc_vacancies(self.h, _ptr(gid), _ptr(site), C.byref(n)))
        return gid[: n.value], site[: n.value]

    def set_world_model(self, tnet, hidden: int, tau_act: float = 1.0):
        """World-model time mode (akmc_set_world_model): policy-logit selection (Eqs. 1-2), Eq. 7 clock."""
        t = np.ascontiguousarray(tnet, dtype=np.float64)
        self._tnet = t
        self._check(self.lib.akmc_set_world_model(self.h, _ptr(t), int(hidden), float(tau_act)))

    def set_dataflow(self, on: bool = True):
        """Dataflow sweeps (akmc_set_dataflow): tiles start a phase when their neighbours finished the previous one."""
        self._check(self.lib.akmc_set_dataflow(self.h, 1 if on else 0))

    def exchange_stats(self) -> dict:
        """Multi-rank: per-phase exchanges, messages and bytes this rank sent."""
        o = np.zeros(3, dtype=np.int64)
        self._check(self.lib.akmc_exchange_stats(self.h, _ptr(o)))
        return {"exchanges": int(o[0]), "messages": int(o[1]), "bytes": int(o[2])}

    def voxel_order(self) -> np.ndarray:
        """Voxel ids in the engine's dispatch order (descending Eq. 10 workload proxy)."""
        o = np.empty(self.cfg.n_voxels, dtype=np.int32)
        self._check(self.lib.akmc_voxel_order(self.h, _ptr(o)))
        return o

    def progress(self):
        """(per-voxel serial event counters, sublattice sweeps done): with state(), a full checkpoint."""
        nev = np.empty(self.cfg.n_voxels, dtype=np.int64)
        sw = C.c_int64(0)
        self._check(self.lib.akmc_progress(self.h, _ptr(nev), C.byref(sw)))
        return nev, int(sw.value)

    def restore(self, vac_sites=None, clock=None, nev=None, sweep: int = 0):
        """Resume a checkpoint on a handle created from its lattice (akmc_restore)."""
        v = None if vac_sites is None else np.ascontiguousarray(vac_sites, dtype=np.int64)
        c = None if clock is None else np.ascontiguousarray(clock, dtype=np.float64)
        n = None if nev is None else np.ascontiguousarray(nev, dtype=np.int64)
        self._check(self.lib.akmc_restore(self.h, _ptr(v), 0 if v is None else int(v.size), _ptr(c), _ptr(n),
                                          int(sweep)))

    def debug_extended(self) -> np.ndarray:
        """Voxel-0 block including its 2-cell halo, canonical over the extended box (diagnostics)."""
        Lx, Ly, Lz = (c + 4 for c in self.cfg.cells)
        out = np.empty(2 * Lx * Ly * Lz, dtype=np.uint8)
        self._check(self.lib.akmc_debug_extended(self.h, _ptr(out)))
        return out

    def rates(self):
        gid, _ = self.vacancies()
        R = np.empty((max(gid.size, 1), 8)); E = np.empty((max(gid.size, 1), 8))
        self._check(self.lib.akmc_rates(self.h, _ptr(R), _ptr(E)))
        return R[: gid.size], E[: gid.size]

    def eval_windows(self, windows, precision: int) -> np.ndarray:
        w = np.ascontiguousarray(windows, dtype=np.uint8).reshape(-1, 64)
        E = np.empty((w.shape[0], 8))
        self._check(self.lib.akmc_eval_windows(self.h, _ptr(w), int(w.shape[0]), int(precision), _ptr(E)))
        return E

    def set_stream(self, stream_ptr: int):
        self._check(self.lib.akmc_set_stream(self.h, C.c_void_p(int(stream_ptr)) if stream_ptr else None))

    def set_voxel_temperatures(self, T_K):
        """Per-voxel temperature in K, one per voxel (C4 variant); clears the barrier memo."""
        t = np.ascontiguousarray(T_K, dtype=np.float64).reshape(-1)
        self._check(self.lib.akmc_set_voxel_temperatures(self.h, _ptr(t), int(t.size)))

    def set_profiling(self, on: bool):
        self._check(self.lib.akmc_set_profiling(self.h, 1 if on else 0))

    def close(self):
        if getattr(self, "h", None):
            self.lib.akmc_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def mfpt_solve(row_ptr, col, rate, tol: float = 1e-13, max_iter: int = 100000):
    """Exact MFPT (Eq. 5) on the device: (tau [n], iterations, relative residual) -- akmc_mfpt_solve."""
    lib = load()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    c = np.ascontiguousarray(col, dtype=np.int32)
    r = np.ascontiguousarray(rate, dtype=np.float64)
    n = rp.size - 1
    tau = np.empty(max(n, 1))
    it = C.c_int32(0)
    res = C.c_double(0.0)
    rc = lib.akmc_mfpt_solve(_ptr(rp), _ptr(c), _ptr(r), int(n), float(tol), int(max_iter), _ptr(tau), C.byref(it),
                             C.byref(res))
    if rc != AKMC_OK:
        raise AkmcError(rc, "akmc_mfpt_solve failed")
    return tau[:n], int(it.value), float(res.value)


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId for Config.nccl_id (call on rank 0, broadcast to the other ranks)."""
    buf = (C.c_uint8 * 128)()
    rc = load().akmc_nccl_unique_id(buf)
    if rc != AKMC_OK:
        raise AkmcError(rc, "ncclGetUniqueId failed")
    return bytes(buf)
