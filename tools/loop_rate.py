#!/usr/bin/env python3
"""Iterations/s of the persistent SPGM loop (nf_spgm_loop) against the CUDA-graph step on a BASELINE workload:
device-sampled flat batches, CUDA events around K iterations.

    python tools/loop_rate.py --workload small --iters 2000
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00774_b200 import configs  # noqa: E402
from paper_2509_00774_b200.plan import DevicePlan  # noqa: E402
from paper_2509_00774_b200.solver import SPGMEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="small")
ap.add_argument("--iters", type=int, default=2000)
ap.add_argument("--dtype", default=None)
ap.add_argument("--batch", type=int, default=None)
a = ap.parse_args()
w = configs.WORKLOADS[a.workload]()
scn = w.scenario
dtype = a.dtype or w.dtype
if a.batch:
    import dataclasses
    w = dataclasses.replace(w, batch=a.batch)
rng = np.random.default_rng(0)
y = rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)
plan = DevicePlan(scn, dtype=dtype, device="cuda:0", max_batch=w.batch)
eng = SPGMEngine(plan, y, eta=1e-3, alpha=1e-7)
st = torch.cuda.current_stream()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


K = a.iters
t_loop = timed(lambda: eng.run_loop(K, table=None, seed=0, iter0=1, batch=w.batch, tol=0.0))
n, reason = eng.loop_result()
g = eng.graph(0, w.batch, pairs=8)
t_graph = timed(lambda: [g.replay() for _ in range(K // 16)]) / (16 * (K // 16)) * K
prof = None
if os.environ.get("NFGPU_LOOP_PROFILE"):
    import ctypes

    per_cta = os.environ["NFGPU_LOOP_PROFILE"] == "2"
    n = K * (12 + (2 * 160 if per_cta else 0)) + (160 if per_cta else 0)
    buf = (ctypes.c_uint64 * n)()
    rc = plan.lib.nf_loop_profile(plan._h, buf, n)
    if rc == 0 and per_cta:  # every CTA's forward / adjoint end relative to CTA 0's phase start
        t0 = np.frombuffer(buf, dtype=np.uint64)[: K * 12].reshape(K, 12).astype(np.float64)
        nsm = torch.cuda.get_device_properties(0).multi_processor_count
        c = np.frombuffer(buf, dtype=np.uint64)[K * 12: K * 332].reshape(K, 2, 160).astype(np.float64)[:, :, :nsm]
        smid = np.frombuffer(buf, dtype=np.uint64)[K * 332: K * 332 + nsm].astype(int)
        sl = slice(K // 4, K - 1)
        fe = (c[sl, 0, :] - t0[sl, 0:1]) / 1e3
        ae = (c[sl, 1, :] - t0[sl, 6:7]) / 1e3
        cta_prof = {"fwd_end_min": fe.min(1).mean(), "fwd_end_mean": fe.mean(), "fwd_end_max": fe.max(1).mean(),
                    "adj_end_min": ae.min(1).mean(), "adj_end_mean": ae.mean(), "adj_end_max": ae.max(1).mean(),
                    "adj_slowest_ctas": np.argsort(-ae.mean(0))[:8].tolist(),
                    "adj_end_by_cta_q": np.percentile(ae.mean(0), [0, 25, 50, 75, 100]).round(2).tolist(),
                    "adj_end_by_cta": ae.mean(0).round(2).tolist(), "fwd_end_by_cta": fe.mean(0).round(2).tolist(),
                    "smid": smid.tolist()}
        print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in cta_prof.items()}))
    if rc == 0:
        t = np.frombuffer(buf, dtype=np.uint64)[: K * 12].reshape(K, 12).astype(np.float64)[K // 4:]
        tiny = not t[:, 6:].any()
        names = (["fwd", "bar0", "sums+adj+prox", "bar1", "stats"] if tiny else
                 ["fwd (next sort first on one CTA)", "bar1", "reduce: partials to shared (stats of k-1 on one CTA)", "reduce: segment sums", "reduce: level 2 + residual records",
                  "bar3", "adj", "bar4"])
        last = 5 if tiny else 8
        d = np.diff(t[:, :last + 1], axis=1).mean(axis=0) / 1e3
        prof = {n: round(float(v), 2) for n, v in zip(names, d)}
        prof["next_iter_gap"] = round(float((t[1:, 0] - t[:-1, last]).mean() / 1e3), 2)
print(json.dumps({"workload": a.workload, "profile_us": prof, "dtype": dtype, "batch": w.batch, "iters": K, "loop_iters_run": n,
                  "loop_us_per_iter": t_loop / K * 1e6, "loop_iters_per_s": K / t_loop,
                  "graph_us_per_iter": t_graph / K * 1e6, "graph_iters_per_s": K / t_graph}))
