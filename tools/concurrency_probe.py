#!/usr/bin/env python3
"""Probe: do two half-batch SPGM pipelines on two streams finish faster than the full batch on one?
Times K steps of (a) one engine at |B| and (b) two engines at |B|/2 each on their own stream,
launched interleaved (eager launches, device sampler). Prints one JSON line per workload.

    python tools/concurrency_probe.py --workload medium --steps 200
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00774_b200 import configs  # noqa: E402
from paper_2509_00774_b200.plan import DevicePlan  # noqa: E402
from paper_2509_00774_b200.solver import SPGMEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="medium")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--zslab", type=int, default=0)
    a = ap.parse_args()
    w = configs.WORKLOADS[a.workload]()
    scn = w.scenario
    rng = np.random.default_rng(0)
    y = (rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)).astype(np.complex64)
    zr = (0, a.zslab) if a.zslab else None
    B = w.batch

    def engine(b):
        p = DevicePlan(scn, dtype=w.dtype, device="cuda:0", max_batch=b, z_range=zr)
        return SPGMEngine(p, y, 1e-2, 1e-6)

    def timed(fn, n):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    full = engine(B)

    def step_full():
        full.sample_device(0, None, B)
        full.step_staged()

    ms_full = timed(step_full, a.steps)
    h1, h2 = engine(B // 2), engine(B // 2)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    main_s = torch.cuda.current_stream()

    def step_two():
        s1.wait_stream(main_s)
        s2.wait_stream(main_s)
        with torch.cuda.stream(s1):
            h1.sample_device(0, None, B // 2)
            h1.step_staged()
        with torch.cuda.stream(s2):
            h2.sample_device(1, None, B // 2)
            h2.step_staged()
        main_s.wait_stream(s1)
        main_s.wait_stream(s2)

    ms_two = timed(step_two, a.steps)

    def step_seq():
        h1.sample_device(0, None, B // 2)
        h1.step_staged()
        h2.sample_device(1, None, B // 2)
        h2.step_staged()

    ms_seq = timed(step_seq, a.steps)
    print(json.dumps({"workload": a.workload, "zslab": a.zslab, "B": B, "full_ms": ms_full,
                      "two_halves_concurrent_ms": ms_two, "two_halves_serial_ms": ms_seq}), flush=True)


if __name__ == "__main__":
    main()
