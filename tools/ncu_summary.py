"""Summarise ncu outputs for profiles/ (run here, on the files gpurun brings back).

  python tools/ncu_summary.py launches <launches.csv> <out_prefix>
      per-kernel launch counts / total / average duration / share from a
      `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list
  python tools/ncu_summary.py full <report.ncu-rep> <out_prefix>
      key metrics, stall reasons and hottest source lines of a `--set full` capture;
      writes <out_prefix>.json (incl. dram_bytes_per_launch) and <out_prefix>.md
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[hi], rows[hi + 1:]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= iv:
            continue
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        agg[r[ik].split("(")[0]][0] += 1
        agg[r[ik].split("(")[0]][1] += v
    tot = sum(v[1] for v in agg.values())
    with open(out + ".csv", "w") as f:
        f.write("kernel,launches,total_ns,avg_ns,share\n")
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f'"{k}",{n},{t:.0f},{t / n:.0f},{t / tot:.4f}\n')
    print(open(out + ".csv").read())


def _ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def full(rep, out):
    raw = list(csv.reader(io.StringIO(_ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    get = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}

    def num(name):
        v, u = get.get(name, ("nan", ""))
        x = float(v.replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
                 "ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6}
        return x * scale.get(u, 1), u
    rd, _ = num("dram__bytes_read.sum")
    wr, _ = num("dram__bytes_write.sum")
    dur, _ = num("gpu__time_duration.sum")
    res = {"report": rep.split("/")[-1], "kernel": get.get("Kernel Name", ("?",))[0],
           "duration_us": dur, "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
           "achieved_dram_GBps": (rd + wr) / (dur * 1e-6) / 1e9 if dur else None}
    for k in ["sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
              "launch__cluster_dim_x" , "smsp__inst_executed.sum",
              # tensor pipe (the barrier network's layers 2-3) and L2 (the gather / W1' rows are L2 traffic)
              "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
              "TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
              "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
              "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
              "lts__t_bytes.sum", "lts__t_sectors_op_read.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
              "l1tex__t_bytes.sum", "sm__cycles_elapsed.avg"]:
        if k in get:
            res[k] = get[k][0]
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(vals[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    res["stall_share"] = {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda x: -x[1]) if v / tot > 0.005}
    # hottest CUDA source lines
    src = list(csv.reader(io.StringIO(_ncu("-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"))))
    cur, lines = None, {}
    for r in src:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or r[0] == "":
            continue
        try:
            lines[(cur, int(r[0]))] = (float(r[4]), r[1].strip()[:90])
        except (ValueError, IndexError):
            pass
    ltot = sum(v[0] for v in lines.values()) or 1.0
    res["hot_lines"] = [{"where": f"{f}:{n}", "share": round(v[0] / ltot, 4), "src": v[1]}
                        for (f, n), v in sorted(lines.items(), key=lambda x: -x[1][0])[:25]]
    json.dump(res, open(out + ".json", "w"), indent=1)
    with open(out + ".md", "w") as f:
        f.write(f"# ncu --set full: {res['kernel']}\n\nreport `{res['report']}` (one launch, cold caches, serialised)\n\n")
        f.write("| metric | value |\n|---|---|\n")
        for k, v in res.items():
            if k not in ("stall_share", "hot_lines"):
                f.write(f"| {k} | {v} |\n")
        f.write("\n## warp stall reasons (share of PC samples)\n\n| reason | share |\n|---|---|\n")
        for k, v in res["stall_share"].items():
            f.write(f"| {k} | {v} |\n")
        f.write("\n## hottest source lines (share of PC samples)\n\n| where | share | source |\n|---|---|---|\n")
        for h in res["hot_lines"]:
            f.write(f"| {h['where']} | {h['share']} | `{h['src'].replace('|', '/')}` |\n")
    print(open(out + ".md").read())


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
