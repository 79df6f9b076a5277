"""bench.py's own arm on the GPU (short runs): the JSON line keeps the driver contract on a serial workload with
batched replicas (--replicas), on the world-model mode (--world) and on the default C5 line's keys."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"}


def _run(*args):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, "bench.py", "--steps", "2", "--warmup", "3", "--ramp-s", "0",
                        "--no-cpu-baseline", *args], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert KEYS <= set(d), KEYS - set(d)
    assert d["value"] > 0 and d["unit"] == "hop-evals/s" and d["gpu_launches"] > 0 and d["n_gpus"] == 1
    for k in ("bound", "achieved", "peak", "frac", "unit"):
        assert k in d["roofline"], k
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    return d


def test_bench_c1_replicas():
    d = _run("--workload", "c1", "--replicas", "256")
    assert d["config"]["voxels_per_gpu"] == 256 and d["config"]["workload"] == "C1"


def test_bench_world_mode():
    d = _run("--workload", "c4", "--world")
    assert d["dtype"] == "f64" and "world-model" in d["config"]["model"]
    assert d["roofline"]["unit"] == "TFLOP/s" and d["roofline"]["rows"] > 0


def test_bench_c3_line():
    d = _run("--workload", "c3")
    assert d["roofline"]["bound"] == "latency" and "evaluator_bulk" in d["roofline"]
    assert d["executed_hop_evals_per_s"] > 0 and d["events_per_s"] > 0
