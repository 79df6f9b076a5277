"""bench.py's reference arm on CPU (-m "not gpu"): the driver runs `bench.py --impl reference` (the oracle as it
stands, a bounded sample of the workload) at N = 1 and under torchrun at N > 1, where rank 0 alone prints the one
JSON line and the other ranks exit 0 without work.  Checks the line's contract keys for a serial workload, for the
world-model mode (--world) and for the 2-process launch."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _lines(out):
    return [json.loads(l) for l in out.splitlines() if l.strip().startswith("{")]


def _check(line, world=False):
    assert KEYS <= set(line), KEYS - set(line)
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "hop-evals/s"
    assert line["higher_is_better"] is True and line["dtype"] == "f64"
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["value"] == line["value"] and cb["sample"]
    assert ("world-model" in cb["sample"]) == world
    e = line["e2e"]
    assert e["value"] == line["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_reference_arm_serial_and_world():
    for extra, world in (([], False), (["--world"], True)):
        r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c1", "--steps", "1",
                            "--warmup", "1", *extra], cwd=ROOT, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        lines = _lines(r.stdout)
        assert len(lines) == 1, r.stdout
        _check(lines[0], world)


def test_reference_arm_under_torchrun_prints_once():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29791", "bench.py", "--impl", "reference",
                        "--workload", "c1", "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1, r.stdout
    _check(lines[0])
    assert lines[0]["n_gpus"] == 2
