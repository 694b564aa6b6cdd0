#!/usr/bin/env python3
"""Aggregate an ncu source page (--page source --csv --print-source cuda,sass) by CUDA source line:
warp-stall samples per line with the top stall reasons, sorted by samples.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > x.csv
    python tools/ncu_lines.py x.csv [--top 40] [--src paper_2509_00774_b200/csrc/nfgpu.cu]
"""
import argparse
import collections
import csv

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--src", default="paper_2509_00774_b200/csrc/nfgpu.cu")
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
hdr = start = None
for i, r in enumerate(rows):
    if r and r[0] == "Line No":
        hdr, start = r, i + 1
        break
reasons = [(j, h) for j, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
per = collections.defaultdict(collections.Counter)
inst = collections.Counter()
line = None
cur = ""
for r in rows[start:]:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1]
        continue
    if not r[0].strip().isdigit() and r[0].strip():
        continue
    if r[0].strip():
        line = int(r[0])
    if not cur.endswith(a.src.split("/")[-1]) and cur:
        continue
    if len(r) < len(hdr) or not r[2].strip():
        continue
    try:
        s = float(r[4] or 0)
    except ValueError:
        continue
    tot[line] += s
    inst[line] += float(r[7] or 0)
    for j, h in reasons:
        per[line][h[6:]] += float(r[j] or 0)
src = open(a.src).read().splitlines()
allS = sum(tot.values())
print(f"total samples {allS:.0f}")
for ln, s in tot.most_common(a.top):
    top = ", ".join(f"{k} {v/s*100:.0f}%" for k, v in per[ln].most_common(3) if v)
    print(f"{ln:5d} {s/allS*100:5.1f}% inst {inst[ln]:10.0f}  {src[ln-1].strip()[:70]:70s} | {top}")
