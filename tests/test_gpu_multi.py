"""Multi-GPU parity (C5 spatial decomposition, halo deltas between phases over NVLink peer memory, NCCL only at init): the same global problem
on 2 ranks and on 1 rank gives bit-identical lattices, vacancy lists, clocks and event counts (GPU-count
invariance, SURVEY 8(c) decomposition pin), and equals the FP64 oracle.  Needs >= 2 GPUs."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("grid,extra", [((2, 1, 1), ["--oracle"]), ((1, 2, 1), []),
                                        ((2, 1, 1), ["--model", "mlp", "--precision", "fp32"]),
                                        ((2, 1, 1), ["--oracle", "--cells", "18", "16", "30", "--domain", "6", "8", "10"])])
def test_two_rank_invariance(tmp_path, grid, extra):
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    out = tmp_path / "multi.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(29600 + grid[1] + 3 * len(extra)), os.path.join(ROOT, "tools", "multi_check.py"),
           "--grid", *map(str, grid), "--out", str(out), *extra]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert res["ok"], res
    assert res["events"] > 20


@pytest.mark.parametrize("grid,extra", [((2, 2, 1), ["--oracle", "--nvac", "60"]), ((1, 2, 2), ["--oracle", "--nvac", "60"]),
                                        ((2, 2, 1), ["--model", "mlp", "--precision", "fp32", "--nvac", "60"]),
                                        ((1, 2, 2), ["--oracle", "--nvac", "60", "--cells", "12", "18", "14",
                                                     "--domain", "6", "6", "14"])])
def test_four_rank_invariance(tmp_path, grid, extra):
    """Two decomposed axes (edge and corner halos, 3 distinct peers per rank): 4 ranks == 1 rank (== oracle)."""
    if _ngpu() < 4:
        pytest.skip("needs 4 GPUs")
    out = tmp_path / "multi4.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=4", "--master-addr",
           "127.0.0.1", "--master-port", str(29670 + grid[0] + 2 * grid[2] + 3 * len(extra)), os.path.join(ROOT, "tools", "multi_check.py"),
           "--grid", *map(str, grid), "--out", str(out), *extra]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert res["ok"], res
    assert res["events"] > 20


@pytest.mark.parametrize("nproc,grid,extra", [(2, (2, 1, 1), ["--oracle"]),
                                              (2, (2, 1, 1), ["--model", "mlp", "--precision", "fp32"]),
                                              (4, (2, 2, 1), ["--oracle", "--nvac", "60"])])
def test_overlapped_exchange_invariance(tmp_path, nproc, grid, extra):
    """AKMC_OVERLAP=1: the receive side of each phase's exchange and the boundary domains' lists run on a second
    stream while the next phase's engine runs the interior domains -- same lattices as 1 rank and the oracle."""
    if _ngpu() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    out = tmp_path / "multi_ov.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}", "--master-addr",
           "127.0.0.1", "--master-port", str(29720 + 7 * nproc + 3 * len(extra)), os.path.join(ROOT, "tools", "multi_check.py"),
           "--grid", *map(str, grid), "--out", str(out), *extra]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env={**os.environ, "AKMC_OVERLAP": "1"})
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert res["ok"], res
    assert res["events"] > 20


def test_two_rank_nccl_transport(tmp_path):
    """SURVEY 4.2 L4 (transport equivalence): the per-phase deltas over NCCL send/recv (AKMC_EXCHANGE=nccl)
    give the same lattices as 1 rank and the oracle, like the default peer-mailbox path above."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    out = tmp_path / "multi_nccl.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", "29641", os.path.join(ROOT, "tools", "multi_check.py"),
           "--grid", "2", "1", "1", "--out", str(out), "--oracle"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, AKMC_EXCHANGE="nccl"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert res["ok"], res
    assert res["events"] > 20


def test_eight_rank_invariance(tmp_path):
    """2x2x2 (all three axes decomposed, 7 distinct peers per rank, corner halos): 8 ranks == 1 rank (== oracle)."""
    if _ngpu() < 8:
        pytest.skip("needs 8 GPUs")
    out = tmp_path / "multi8.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8", "--master-addr",
           "127.0.0.1", "--master-port", "29688", os.path.join(ROOT, "tools", "multi_check.py"),
           "--grid", "2", "2", "2", "--out", str(out), "--oracle", "--nvac", "120"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert res["ok"], res
    assert res["events"] > 20


def test_two_rank_slot_reuse_long_run(tmp_path):
    """departed local slots are reused by arrivals (akmc_dist.cuh FreeList).  With the spare slot
    capacity shrunk to 4 (AKMC_VCAP_SPARE) a long run migrates far more vacancies than the spare holds; it must
    neither overflow nor change the trajectory (2 ranks == 1 rank == oracle)."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    out = tmp_path / "multi_reuse.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", "29653", os.path.join(ROOT, "tools", "multi_check.py"),
           "--grid", "2", "1", "1", "--out", str(out), "--oracle", "--sweeps", "60", "--cells", "12", "12", "12",
           "--domain", "6", "6", "6", "--nvac", "30"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, AKMC_VCAP_SPARE="4"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert res["ok"], res
    assert res["events"] > 200


@pytest.mark.parametrize("grid,nproc,direct_msgs,shift_msgs", [((2, 1, 1), 2, 1, 1), ((2, 2, 1), 4, 3, 2),
                                                              ((1, 2, 2), 4, 3, 2), ((2, 2, 2), 8, 7, 3)])
def test_shift_exchange_equals_direct(tmp_path, grid, nproc, direct_msgs, shift_msgs):
    """S:766 / P:420-427: the per-phase deltas by shift communication (X -> Y -> Z stages, AKMC_EXCHANGE=shift)
    give the same global lattice, vacancies and clocks as 1 rank and the oracle -- as the direct exchange does --
    with fewer messages per rank and phase (2x2x1: 2 vs 3 distinct peers; 2x2x2: 3 vs 7)."""
    if _ngpu() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    res = {}
    for mode in ("shift", "p2p"):
        out = tmp_path / f"multi_{mode}.json"
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}", "--master-addr",
               "127.0.0.1", "--master-port", str(29710 + grid[0] + 3 * grid[1] + 7 * grid[2] + (mode == "p2p")),
               os.path.join(ROOT, "tools", "multi_check.py"), "--grid", *map(str, grid), "--out", str(out), "--oracle",
               "--nvac", str(30 * nproc)]
        r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                           env=dict(os.environ, AKMC_EXCHANGE=mode))
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        res[mode] = json.loads(out.read_text())
        assert res[mode]["ok"], res[mode]
        assert res[mode]["events"] > 20
    assert res["shift"]["events"] == res["p2p"]["events"]
    assert all(m == shift_msgs for m in res["shift"]["messages_per_phase"]), res["shift"]["messages_per_phase"]
    assert all(m == direct_msgs for m in res["p2p"]["messages_per_phase"]), res["p2p"]["messages_per_phase"]
