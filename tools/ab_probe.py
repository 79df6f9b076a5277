"""A/B timing of library variants on one box (diagnostic, GPU).

  python tools/ab_probe.py NAME=path/to/lib.so [NAME=...] [--cells 1024] [--sweeps 4] [--reps 2]

Runs tools/iter_probe.py once per (rep, variant) in a fresh process with AKMC_LIB pointing at the variant,
alternating variants, and prints the median host-stepped wall ms per sweep (sweeps after the first) and
the event counts (identical across variants when a change is bit-preserving).
"""
import json
import os
import statistics
import subprocess
import sys


def main():
    args = [a for a in sys.argv[1:] if "=" in a and not a.startswith("--")]
    rest = [a for a in sys.argv[1:] if a not in args]
    reps = 2
    if "--reps" in rest:
        i = rest.index("--reps"); reps = int(rest[i + 1]); del rest[i:i + 2]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for r in range(reps):
        for a in args:
            name, path = a.split("=", 1)
            env = dict(os.environ, AKMC_LIB=os.path.abspath(path))
            out = subprocess.run([sys.executable, os.path.join(root, "tools", "iter_probe.py"), "--no-rates", *rest],
                                 env=env, capture_output=True, text=True, timeout=600)
            rows = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{\"sweep\"")]
            res.setdefault(name, []).append(rows)
            for l in out.stderr.splitlines():
                if l.startswith("[akmc engine]") or l.startswith("[akmc iter trace]"):
                    print(f"{name} rep{r} {l}")
            print(name, r, [round(x["wall_ms"], 3) for x in rows], [x["events"] for x in rows], flush=True)
    for name, runs in res.items():
        ms = [x["wall_ms"] for rows in runs for x in rows[1:]]
        print(f"== {name}: median {statistics.median(ms):.3f} ms/sweep over {len(ms)} sweeps; events "
              f"{[x['events'] for x in runs[0]]}")


if __name__ == "__main__":
    main()
