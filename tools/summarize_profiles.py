#!/usr/bin/env python3
"""Regenerate profiles/<round>_ncu_summary.json (base units: bytes, ns, cycles/s) and the measured tables of
profiles/<round>_summary.md from the committed bench JSON lines, the peaks JSON, the launch
list and an ncu --set full report (read here with `ncu -i`; the .ncu-rep itself is scratch).

    python tools/summarize_profiles.py --round r01 --ncu gpurun_out/prof.ncu-rep
"""
import argparse
import csv
import json
import subprocess
from collections import defaultdict
from pathlib import Path

P = Path(__file__).resolve().parents[1] / "profiles"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second"]
STALLS = ["wait", "short_scoreboard", "long_scoreboard", "math_pipe_throttle", "mio_throttle", "not_selected"]


def ncu_summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    out = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        d = {k: float(r[h.index(k)].replace(",", "")) for k in KEYS if k in h and r[h.index(k)]}
        for st in STALLS:
            k = f"smsp__average_warps_issue_stalled_{st}_per_issue_active.ratio"
            if k in h:
                d["stall_" + st] = float(r[h.index(k)])
        out[name] = d
    return out


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            d[r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:44]].append(float(r[vi]))
    tot = sum(sum(v) for v in d.values())
    lines = ["| kernel | launches | mean µs/launch | share |", "|---|---|---|---|"]
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.1%} |")
    return "\n".join(lines)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--ncu", required=True)
    a = ap.parse_args()
    s = ncu_summary(a.ncu)
    json.dump(s, open(P / f"{a.round}_ncu_summary.json", "w"), indent=1)
    print(json.dumps(s, indent=1)[:3000])
    print(launch_table(P / f"{a.round}_launches.csv"))


if __name__ == "__main__":
    main()
