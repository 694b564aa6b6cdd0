#!/usr/bin/env python3
"""BASELINE config 5, the operator microbenchmark: one forward A s and one adjoint A^H r at full M
(64 Tx x 64 Rx x 256 f = 1,048,576 channels) on the 64³, 128³ and 192x192x96 grids, random N(0,1)
complex inputs, CUDA events, one warm-up run each.

Full M is a Cartesian product, so it is timed twice: through the flat kernels (nf_batch_prepare
with the channel list) and through the separable kernels (nf_batch_prepare_structured). The two
results are compared (relative L2). One JSON line per (grid, dtype).

    python tools/microbenchmark.py [--grids 64^3,128^3,192x192x96] [--c128-grids 64^3]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2509_00774_b200 import configs  # noqa: E402
from paper_2509_00774_b200.plan import DevicePlan  # noqa: E402


def timed(fn, warm: bool = True):
    if warm:
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.current_stream()
    e0.record(st)
    out = fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3, out


def rel(a, b):
    return float(torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b))


def run(grid: str, dtype: str, paths=("flat", "structured")):
    """One full-M forward and adjoint per path. c128 operations last seconds, so they are timed on
    their first call (no warm-up run: kernel attributes and first-launch costs are microseconds)."""
    scn = configs.micro_scenario(grid)
    plan = DevicePlan(scn, dtype=dtype)
    M, N = scn.n_channels, scn.n_voxels
    g = torch.Generator(device=plan.device).manual_seed(3)
    cd = plan.torch_dtype
    s = torch.randn(N, dtype=cd, device=plan.device, generator=g)
    r = torch.randn(M, dtype=cd, device=plan.device, generator=g)
    y = plan.vec(M)
    z = plan.vec(N)
    out = {"grid": grid, "dtype": dtype, "M": M, "N": N, "entries_per_op": M * N}
    res = {}
    warm = dtype == "c64"
    for path in paths:
        if path == "flat":
            plan.prepare(torch.arange(M, dtype=torch.int32, device=plan.device))
        else:
            plan.prepare_full()
        tf, yv = timed(lambda: plan.forward(s, out=y).clone(), warm)
        ta, zv = timed(lambda: plan.adjoint(r, out=z).clone(), warm)
        res[path] = (yv, zv)
        out[path] = {"fwd_s": tf, "adj_s": ta, "fwd_entries_per_s": M * N / tf, "adj_entries_per_s": M * N / ta}
    if len(res) == 2:
        out["structured_vs_flat_rel_l2"] = {"forward": rel(res["structured"][0], res["flat"][0]),
                                            "adjoint": rel(res["structured"][1], res["flat"][1])}
    del plan, res
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grids", default="64^3,128^3,192x192x96")
    ap.add_argument("--c128-grids", default="64^3")
    a = ap.parse_args()
    for grid in a.grids.split(","):
        print(json.dumps(run(grid, "c64")), flush=True)
        torch.cuda.empty_cache()
    for grid in filter(None, a.c128_grids.split(",")):
        print(json.dumps(run(grid, "c128")), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
