"""Build the sm_100a shared library libakmc.so in-tree (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libakmc.so")
SOURCES = ["akmc_api.cu", "akmc_engine.cu", "akmc_bulk.cu", "akmc_world.cu", "akmc_mfpt.cu"]
HEADERS = ["akmc_world.cuh", "akmc_eval.cuh", "akmc_device.cuh", "akmc_kernels.cuh", "akmc_dist.cuh", "akmc_p2p.cuh", "akmc_engine.cuh", "akmc_ptx.cuh"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2"]


def nccl_flags() -> list:
    """NCCL from the wheel torch uses (same libnccl.so.2 in-process), else the system one."""
    import glob
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        root = list(spec.submodule_search_locations)[0]
        inc, lib = os.path.join(root, "include"), os.path.join(root, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and glob.glob(os.path.join(lib, "libnccl.so*")):
            return ["-I" + inc, "-L" + lib, "-l:libnccl.so.2", "-Xlinker", "-rpath," + lib]
    return ["-lnccl"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "akmc.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines: tuple = ()) -> str:
    """Build LIB (or `out`, an A/B variant compiled with extra -D `defines`)."""
    target = out or LIB
    if not force and not defines and target == LIB and not _stale():
        return LIB
    os.makedirs(os.path.dirname(target), exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = target + ".tmp"
    cmd = [nvcc, *NVCC_FLAGS, *["-D" + d for d in defines], *[os.path.join(CSRC, s) for s in SOURCES], *nccl_flags(),
           "-o", tmp]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force=True, verbose=True))
