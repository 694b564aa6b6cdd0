#!/usr/bin/env python3
"""Benchmark of the SPGM hot path (BASELINE.json metric: A-entry evals/s, fwd+adj,
and SPGM iterations/s, as a fraction of the FP32+SFU roofline).

One step = one SPGM iteration on the chosen workload (default: BASELINE 'Large',
|B| = 4096 flat minibatch, complex64): device sampler → batch prepare → fused
forward → [NCCL all-reduce of the 2·|B| partial sums over voxel slabs] → fused
adjoint + soft-threshold prox + termination statistics. Entries per step = 2·|B|·N.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload large|medium|small]
    python bench.py --impl reference ...   # the reference algorithm on the host CPU

N > 1 runs under torchrun (one process per GPU, voxel-slab sharding, strong scaling).
Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "A-entry evals/sec (fwd+adj) & SPGM iters/sec; % of FP32+SFU roofline, 1/2/4/8 GPU"
UNIT = "entries/s"
# SFU roofline: 2 MUFU (sin, cos) per entry, 16 MUFU/clk/SM, 148 SMs
ENTRIES_PER_CLK_SM = 8.0
N_SM = 148
# measured on this pool's B200 with tools/peaks.cu (profiles/r01_peaks.json): 4.622e12 MUFU sin/cos
# ops/s at 1965 MHz = 15.89 per clk per SM -> 2.311e12 entries/s
SFU_ENTRY_PEAK_MEASURED = 4.622e12 / 2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="large", choices=["large", "medium", "small"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU baseline sample budget")
    ap.add_argument("--no-graph", action="store_true", help="launch steps eagerly instead of a CUDA graph")
    ap.add_argument("--no-extras", action="store_true", help="skip the extra workload lines")
    ap.add_argument("--quick", action="store_true", help="skip the sweep, microbenchmark and full-grid CPU lines")
    ap.add_argument("--cpu-child", default=None, choices=["small", "medium"],
                    help=argparse.SUPPRESS)  # internal: one full-grid CPU baseline in a child process
    ap.add_argument("--force-dist", action="store_true", help="use the distributed path even at world size 1")
    ap.add_argument("--collective", default="auto", choices=["auto", "nccl", "peer"],
                    help="forward-partial all-reduce at N > 1: the fused NVLink peer all-reduce "
                         "(nf_forward_allreduce, DESIGN.md §5), NCCL, or auto = peer when its start-up check "
                         "against NCCL passes on every rank, else NCCL")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 100 ms during the timed region
    (one persistent `nvidia-smi -lms 100` process)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.rows = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.15)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.05)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in out.splitlines():
            cols = [c.strip() for c in line.split(",")]
            if len(cols) == 7:
                self.rows.append(cols)

    def summary(self):
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [v for v in (num(r[0]) for r in self.rows) if v is not None]
        mx = [v for v in (num(r[1]) for r in self.rows) if v is not None]
        pw = [v for v in (num(r[2]) for r in self.rows) if v is not None]
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(sm), "power_w_max": max(pw) if pw else None}


# ---------------------------------------------------------------- CPU baseline (oracle port)


def cpu_baseline(workload: str, steps: int, budget_s: float, rank_sample_seed: int = 0):
    """The reference's CPU algorithm (phasor tables + BLAS dots, forward.py:183-336),
    restated in oracle/ and run with all host threads on a voxel sample of the same
    workload: the whole grid when its tables fit (<= 131072 voxels), else z-plane 0, with the
    same |B| and flat sampling."""
    from oracle import nfmimo_oracle as O
    from paper_2509_00774_b200 import configs

    w = configs.WORKLOADS[workload]()
    geo_full = O.geom_from_scenario(w.scenario) if w.scenario.n_voxels <= 1 << 17 else None
    if geo_full is None:
        v = w.scenario.voxels
        cen = O.centers_of(v.corner.as_array(), v.spacing, v.dims, (0, 1))
        n_sample = cen.shape[0]
        freqs = w.scenario.frequencies.values()
        geo = O.Geom(w.scenario.array.tx_positions(), w.scenario.array.rx_positions(), freqs,
                     w.scenario.pulse.evaluate(freqs), cen, w.scenario.c)
        scn = w.scenario
        full_tables = 16 * scn.frequencies.count * (scn.array.n_tx + scn.array.n_rx) * scn.n_voxels
        sample = (f"z-plane 0 ({n_sample} of {scn.n_voxels} voxels) of the {workload} grid, all M channels "
                  f"(the full grid's phasor tables would need {full_tables / 1e9:.0f} GB)")
    else:
        geo = geo_full
        sample = f"full {workload} grid ({geo.N} voxels)"
    threads = O.host_threads()
    t0 = time.perf_counter()
    op = O.TableOperator(geo)
    build_s = time.perf_counter() - t0
    rng = np.random.default_rng(0)
    y = rng.standard_normal(geo.M) + 1j * rng.standard_normal(geo.M)
    s = np.zeros(geo.N, dtype=np.complex128)
    seq_rng = np.random.default_rng(configs.SEEDS["minibatch"])
    done, t_iter = 0, 0.0
    times = []
    while done < max(steps, 1) and (t_iter < budget_s or done < 2):
        idx = np.sort(seq_rng.choice(geo.M, w.batch, replace=False))
        t1 = time.perf_counter()
        resid = op.forward(s, idx, threads) - y[idx]
        g = op.adjoint(resid, idx, threads) / idx.size
        s = O.soft_threshold(s - 1e-3 * g, 1e-6)
        dt = time.perf_counter() - t1
        times.append(dt)
        t_iter += dt
        done += 1
    per = float(np.mean(times[1:] if len(times) > 2 else times))
    entries = 2.0 * w.batch * geo.N
    return {
        "value": entries / per, "unit": UNIT, "cores": threads, "kind": "port",
        "sample": f"{sample}; |B|={w.batch} flat; {done} SPGM iterations of the oracle's table restatement "
                  f"of the reference algorithm (forward.py:183-336); table build {build_s:.1f}s excluded",
        "iters_timed": done, "s_per_iter": per, "table_build_s": build_s,
        "table_bytes": O.TableOperator.table_bytes(geo),
    }


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    cb = cpu_baseline(args.workload, args.steps, args.cpu_seconds * max(1, args.steps) / 30.0)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": cb["iters_timed"], "warmup": 1, "ms_per_step": cb["s_per_iter"] * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": args.workload, "sample": cb["sample"]},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm


def slab(nz: int, rank: int, world: int):
    from paper_2509_00774_b200.sharding import slab_range

    return slab_range(nz, rank, world)


def build_engine(workload, dev, rank, world, pg, collective="nccl"):
    """Setup (not timed): plan for this rank's slab, synthetic scene and measurements, the
    power-iteration Lipschitz constant (20 iterations, as BASELINE.json), λ and α."""
    from paper_2509_00774_b200 import configs
    from paper_2509_00774_b200.plan import DevicePlan
    from paper_2509_00774_b200.sharding import ShardedSetup
    from paper_2509_00774_b200.solver import SPGMEngine

    w = configs.WORKLOADS[workload]()
    scn = w.scenario
    zr = slab(scn.voxels.dims[2], rank, world)
    t0 = time.perf_counter()
    setup = ShardedSetup(scn, dtype=w.dtype, device=dev, z_range=zr, process_group=pg)
    clean = setup.forward_full(configs.make_scene(w))
    y = configs.add_noise(clean, configs.noise_sigma(clean, w.snr_db))
    L = setup.lipschitz(n_iters=20, rng_seed=configs.SEEDS["power"])
    lam = 1e-3 * setup.max_abs_adjoint(y) / scn.n_channels
    eta, alpha = 1.0 / L, lam / L
    setup.release()
    plan = DevicePlan(scn, dtype=w.dtype, device=dev, z_range=zr, max_batch=w.batch)
    eng = SPGMEngine(plan, y, eta, alpha, process_group=pg, collective=collective)
    return w, plan, eng, eta, alpha, time.perf_counter() - t0


def timed_steps(eng, plan, w, steps, warmup, pg, local, use_graph, clk=None):
    """W untimed + K timed SPGM iterations (device sampler); CUDA events on the launching
    stream, barrier + synchronize on both sides, max over ranks. Returns (ms, launches/step, K)."""
    import torch
    import torch.distributed as dist

    from paper_2509_00774_b200 import configs

    seed, B = configs.SEEDS["minibatch"], w.batch
    l0 = plan.info()["launches"]
    eng.sample_device(seed, None, B)
    eng.step_staged()
    per_step = plan.info()["launches"] - l0
    graph = eng.graph(seed, B, pairs=1) if use_graph else None

    def run(n):
        if graph is not None:
            for _ in range((n + 1) // 2):
                graph.replay()
            return 2 * ((n + 1) // 2)
        for _ in range(n):
            eng.sample_device(seed, None, B)
            eng.step_staged()
        return n

    run(max(warmup, 3))
    torch.cuda.synchronize()
    if pg is not None:
        dist.barrier(device_ids=[local])
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if clk is not None:
        clk.__enter__()
    e0.record(st)
    done = run(steps)
    e1.record(st)
    torch.cuda.synchronize()
    if clk is not None:
        clk.__exit__()
    if pg is not None:
        dist.barrier(device_ids=[local])
    ms = e0.elapsed_time(e1)
    if pg is not None:
        t = torch.tensor([ms], device=plan.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms, per_step, done


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1 or args.force_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
        pg = dist.group.WORLD
    w, plan, eng, eta, alpha, setup_s = build_engine(args.workload, dev, rank, world, pg, args.collective)
    scn = w.scenario
    B, N, M = w.batch, scn.n_voxels, scn.n_channels
    use_graph = not args.no_graph
    clk = ClockSampler(local)
    ms, per_step, steps = timed_steps(eng, plan, w, args.steps, args.warmup, pg, local, use_graph, clk)
    change = eng.magnitude_change()
    ms_step = ms / steps
    value = 2.0 * B * N / (ms_step * 1e-3)

    # per-kernel timing of the two fused kernels (same stream, CUDA events, steady state)
    from paper_2509_00774_b200 import configs

    kt = kernel_times(eng, plan, configs.SEEDS["minibatch"], 10_000, reps=max(5, min(args.steps, 20)))
    if pg is not None:
        t = torch.tensor([kt["fwd_ms"], kt["adj_ms"]], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        kt["fwd_ms"], kt["adj_ms"] = (float(v) for v in t.tolist())

    # e2e: public-API semantics, host buffers: host-sampled indices (numpy, as the reference)
    # H2D each step, the termination statistic D2H each step
    e2e = None
    if not args.no_e2e:
        e2e = e2e_public_api(w, eng, args) if pg is None else e2e_run(eng, scn, B, N, args, pg, local)
    clocks = clk.summary()
    peak = SFU_ENTRY_PEAK_MEASURED
    dom = "adjoint_prox" if kt["adj_ms"] >= kt["fwd_ms"] else "forward"
    dom_ms = max(kt["adj_ms"], kt["fwd_ms"])
    per_launch = B * plan.n_local
    achieved = per_launch / (dom_ms * 1e-3)
    clk = clocks.get("sm_mhz") or 1965.0
    roof = {
        "bound": "fp32+sfu", "kernel": dom, "achieved": achieved / 1e9, "peak": peak / 1e9, "unit": "Gentry/s",
        "frac": achieved / peak,
        "peak_source": "measured MUFU sin/cos rate on this pool's B200 (tools/peaks.cu, profiles/r01_peaks.json): "
                       "15.89 MUFU/clk/SM x 148 SM x 1.965 GHz / 2 MUFU per entry; MEASURED_PEAKS.json has no SFU "
                       "figure; nominal 2326.6 Gentry/s",
        "frac_at_observed_clock": achieved / (peak * clk / 1965.0),
        "fwd_ms": kt["fwd_ms"], "adj_ms": kt["adj_ms"], "entries_per_launch": per_launch,
        "frac_forward": per_launch / (kt["fwd_ms"] * 1e-3) / peak,
        "frac_adjoint_prox": per_launch / (kt["adj_ms"] * 1e-3) / peak,
        "frac_step": value / (world * peak),
        "traffic": ncu_traffic(dom),
        "bound_note": "BASELINE north_star: the operator is generated, not stored, and not a dense contraction, so "
                      "the roofline is the FP32 FMA + MUFU (SFU) pipe (2 MUFU per entry); neither 'hbm' nor "
                      "'tensor' applies (see hbm_view)",
    }
    tr = roof["traffic"]
    if tr is not None:
        peak_hbm = hbm_peak_gbs()
        gbs = tr["bytes_per_launch"] / (dom_ms * 1e-3) / 1e9
        roof["hbm_view"] = {"achieved": gbs, "peak": peak_hbm, "unit": "GB/s",
                            "frac": gbs / peak_hbm if peak_hbm else None,
                            "how": "ncu DRAM bytes per launch of the dominant kernel / its CUDA-event time; peak from "
                                   "MEASURED_PEAKS.json (else the B200_PROFILING.md fallback)"}
    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c64" if w.dtype == "c64" else "c128",
            "data": "synthetic (seeded scene/array/noise with the BASELINE shapes; no dataset)",
            "iters_per_s": 1e3 / ms_step,
            "config": {"workload": args.workload, "M": M, "N": N, "batch": B, "sampler": "device flat (Feistel)",
                       "parallelism": f"voxel-slab x{world}", "collective": eng.collective, "l2": "inputs larger than L2 (distance table "
                       f"{plan.info()['device_bytes'] / 2**30:.2f} GiB streamed per kernel)",
                       "cuda_graph": use_graph, "eta": eta, "alpha": alpha, "setup_s": setup_s},
            "roofline": roof, "clocks": clocks, "gpu_launches": per_step * steps, "launches_per_step": per_step,
            "final_change": change,
        }
        if e2e is not None:
            out["e2e"] = e2e
        if world == 1 and not args.no_extras and args.workload == "large":
            ex = {"medium": medium_line(args, dev), "small": medium_line(args, dev, "small"),
                  "large_structured": structured_line(eng, w), "large_c128": large_c128_line(eng, w, args)}
            if not args.quick:
                ex["minibatch_sweep"] = sweep_line(eng, w)
                ex["microbenchmark"] = micro_lines()
            out["extra_workloads"] = ex
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline(args.workload, 30, args.cpu_seconds)
            out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            if not args.quick and args.workload == "large":
                out["cpu_baseline"]["full_grid"] = {wl: cpu_child(wl) for wl in ("small", "medium")}
        print(json.dumps(out), flush=True)
    if pg is not None:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    return 0


def medium_line(args, dev, workload="medium"):
    """BASELINE config 1 (Medium, |B| = 512, c64) -- or config 0 (Small, |B| = 32, c128) -- on the same GPU:
    entries/s and iterations/s."""
    import torch

    w, plan, eng, eta, alpha, setup_s = build_engine(workload, dev, 0, 1, None)
    ms, per_step, steps = timed_steps(eng, plan, w, 200, 10, None, 0, not args.no_graph)
    N = w.scenario.n_voxels
    out = {"value": 2.0 * w.batch * N / (ms / steps * 1e-3), "unit": UNIT, "ms_per_step": ms / steps,
           "iters_per_s": 1e3 * steps / ms, "steps": steps, "batch": w.batch, "N": N, "M": w.scenario.n_channels,
           "frac_step": 2.0 * w.batch * N / (ms / steps * 1e-3) / SFU_ENTRY_PEAK_MEASURED, "cuda_graph": not args.no_graph,
           "launches_per_step": per_step}
    # the persistent device loop (nf_spgm_loop: one cooperative launch for K iterations, device sampler)
    K = 2000 if workload == "small" else 400
    st = torch.cuda.current_stream()
    eng.run_loop(16, table=None, seed=0, iter0=1, batch=w.batch, tol=0.0)
    eng.loop_result()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    eng.run_loop(K, table=None, seed=0, iter0=17, batch=w.batch, tol=0.0)
    e1.record(st)
    torch.cuda.synchronize()
    n_run, _ = eng.loop_result()
    ms_l = e0.elapsed_time(e1) / n_run
    out["persistent_loop"] = {"value": 2.0 * w.batch * N / (ms_l * 1e-3), "unit": UNIT, "ms_per_step": ms_l,
                              "iters_per_s": 1e3 / ms_l, "iterations": n_run, "launches": 1,
                              "kernel": "tiny_loop_kernel" if w.batch * plan.n_local <= (1 << 20) else "spgm_loop_kernel",
                              "frac_step": 2.0 * w.batch * N / (ms_l * 1e-3) / SFU_ENTRY_PEAK_MEASURED}
    # the line's own numbers are those of the path spgm_solve runs for this config (the persistent loop); the
    # per-iteration step in a CUDA graph stays beside them
    out["cuda_graph_step"] = {k: out[k] for k in ("value", "ms_per_step", "iters_per_s", "steps", "frac_step",
                                                  "launches_per_step")}
    for k in ("value", "ms_per_step", "iters_per_s", "frac_step"):
        out[k] = out["persistent_loop"][k]
    out["path"] = "persistent device loop (nf_spgm_loop), the path spgm_solve runs for this config"
    out.pop("launches_per_step", None)
    out.pop("cuda_graph", None)
    # end to end through spgm_solve (the reference's entry point), host numpy sampling as the reference, the
    # config's own iteration count, y on the host, the final volume back (median of 3 solves after a warm-up)
    from paper_2509_00774_b200.solver import SolverConfig, spgm_solve

    y_host = eng.y.to(torch.complex128).cpu().numpy()
    cfg = SolverConfig(eta=eta, alpha=alpha, max_iters=w.iters, tol=1e-300, dtype=w.dtype, flat_batch=w.batch,
                       rng_seed=configs_seed())
    spgm_solve(y_host, w.scenario, cfg)
    walls = []
    for _ in range(3):
        t0 = time.perf_counter()
        rep = spgm_solve(y_host, w.scenario, cfg)
        walls.append(time.perf_counter() - t0)
    wall = float(np.median(walls))
    out["e2e"] = {"value": 2.0 * w.batch * N * rep.iterations / wall, "unit": UNIT, "iters_per_s": rep.iterations / wall,
                  "wall_s": wall, "iterations": rep.iterations, "h2d_bytes_per_step": 4 * w.batch,
                  "d2h_bytes_per_step": 6 * 8,
                  "how": "wall clock around spgm_solve with the config's iteration count (host numpy flat sampling, the "
                         "reference's call sequence; index tables H2D per chunk of 4..256 iterations, statistics D2H "
                         "per chunk, one IterationRecord per iteration; chained persistent-loop launches)"}
    return out


def configs_seed() -> int:
    from paper_2509_00774_b200 import configs

    return configs.SEEDS["minibatch"]


def structured_line(eng, w):
    """The reference's own minibatch sampler (solver.sample_minibatch: a sorted Cartesian
    n_f × n_tx × n_rx product, solver.py:205-225) on Large through the separable kernels
    (nf_batch_prepare_structured): composition 4 × 32 × 32 = 4096 channels, host-sampled each
    step like the reference, plus the full-batch proximal-gradient (ISTA, |B| = M) step."""
    import torch

    from paper_2509_00774_b200 import configs
    from paper_2509_00774_b200.plan import DevicePlan
    from paper_2509_00774_b200.solver import MinibatchComposition, SPGMEngine, sample_minibatch

    scn = w.scenario
    N, M = scn.n_voxels, scn.n_channels
    st = torch.cuda.current_stream()

    def timed(fn, warm, reps):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    comp = MinibatchComposition(4, 32, 32)
    rng = np.random.default_rng(configs.SEEDS["minibatch"])

    def spgm_step():
        eng.stage(sample_minibatch(comp, scn, rng).indices)
        eng.step_staged()

    ms = timed(spgm_step, 5, 100)
    B = comp.n_f * comp.n_tx * comp.n_rx
    out = {"composition": [comp.n_f, comp.n_tx, comp.n_rx], "batch": B, "structured": eng.plan.staged_structured,
           "value": 2.0 * B * N / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "iters_per_s": 1e3 / ms,
           "sampler": "host numpy (reference sample_minibatch), indices uploaded every step"}
    # the same compositions drawn on the device (nf_sample_structured), 2 steps per CUDA graph replay
    g = eng.graph(configs.SEEDS["minibatch"], 0, pairs=1, composition=comp)
    ms_g = timed(g.replay, 3, 50) / 2
    out["device_sampler_cuda_graph"] = {"value": 2.0 * B * N / (ms_g * 1e-3), "unit": UNIT, "ms_per_step": ms_g,
                                        "iters_per_s": 1e3 / ms_g}
    pf = DevicePlan(scn, dtype=w.dtype, device=eng.plan.device, max_batch=M)
    ef = SPGMEngine(pf, eng.y, eng.eta, eng.alpha, initial=eng.s)
    ef.stage(np.arange(M))
    ms_full = timed(ef.step_staged, 1, 3)
    out["ista_full_batch"] = {"batch": M, "structured": pf.staged_structured, "value": 2.0 * M * N / (ms_full * 1e-3),
                              "unit": UNIT, "ms_per_step": ms_full}
    del ef, pf
    torch.cuda.empty_cache()
    return out


def large_c128_line(eng, w, args):
    """The Large step in complex128, the reference's own precision (and the CPU arm's): same y, eta, alpha,
    |B| = 4096 flat device-sampled batches, CUDA graph, so the like-for-like GPU/CPU ratio is measured."""
    import torch

    from paper_2509_00774_b200.plan import DevicePlan
    from paper_2509_00774_b200.solver import SPGMEngine

    plan = DevicePlan(w.scenario, dtype="c128", device=eng.plan.device, max_batch=w.batch)
    e = SPGMEngine(plan, eng.y.to(torch.complex128), eng.eta, eng.alpha)
    ms, per_step, steps = timed_steps(e, plan, w, 20, 3, None, 0, not args.no_graph)
    N = w.scenario.n_voxels
    v = 2.0 * w.batch * N / (ms / steps * 1e-3)
    out = {"dtype": "c128", "value": v, "unit": UNIT, "ms_per_step": ms / steps, "iters_per_s": 1e3 * steps / ms,
           "steps": steps, "batch": w.batch, "frac_step_sfu_roof": v / SFU_ENTRY_PEAK_MEASURED}
    del e, plan
    torch.cuda.empty_cache()
    return out


def sweep_line(eng, w):
    """BASELINE config 3: the minibatch sweep on Large (|B| in {256 ... 65536} flat, plus ISTA with |B| = M on the
    separable kernels), 100 iterations each from s = 0, device time; objective D(s) + lambda ||s||_1 against
    device time at 25-iteration checkpoints (full-M forward, untimed). tools/minibatch_sweep.py."""
    import torch

    sys.path.insert(0, str(ROOT / "tools"))
    from minibatch_sweep import sweep

    y = eng.y.to(torch.complex128).cpu().numpy()
    summary, _ = sweep(w.scenario, y, eng.eta, eng.alpha, eng.alpha / eng.eta, iters=100, every=25,
                       dev=eng.plan.device)
    return summary


def micro_lines():
    """BASELINE config 4: one full-M forward and one full-M adjoint (M = 64 x 64 x 256) on the 64^3, 128^3 and
    192x192x96 grids, c64 and c128, flat and separable kernels (tools/microbenchmark.py)."""
    sys.path.insert(0, str(ROOT / "tools"))
    from microbenchmark import run

    out = []
    for dtype in ("c64", "c128"):
        for grid in ("64^3", "128^3", "192x192x96"):
            line = run(grid, dtype)
            for path in ("flat", "structured"):
                line[path]["frac_sfu_roof"] = {k: line[path][k] / SFU_ENTRY_PEAK_MEASURED
                                               for k in ("fwd_entries_per_s", "adj_entries_per_s")}
            out.append(line)
    return out


def cpu_child(workload: str) -> dict:
    """Full-grid CPU baseline of one config in a child process, so that its peak RSS (the
    reference's phasor tables, forward.py:190-211) is its own."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--cpu-child", workload]
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        return json.loads(res.stdout.strip().splitlines()[-1])
    except Exception as e:  # reported, not fatal: the GPU line stands on its own
        return {"error": f"{type(e).__name__}: {e}"}


def _vm_hwm_bytes() -> int:
    """Peak resident set of this process (VmHWM; ru_maxrss would carry the forking parent's peak)."""
    for line in open("/proc/self/status"):
        if line.startswith("VmHWM:"):
            return int(line.split()[1]) * 1024
    return -1


def _vm_rss_bytes() -> int:
    for line in open("/proc/self/status"):
        if line.startswith("VmRSS:"):
            return int(line.split()[1]) * 1024
    return -1


def cpu_child_main(workload: str, budget_s: float) -> int:
    from oracle import nfmimo_oracle as O
    from paper_2509_00774_b200 import configs

    w = configs.WORKLOADS[workload]()
    geo = O.geom_from_scenario(w.scenario)
    threads = O.host_threads()
    rss0 = _vm_rss_bytes()
    t0 = time.perf_counter()
    op = O.TableOperator(geo)
    build_s = time.perf_counter() - t0
    rss_tables = _vm_rss_bytes()
    rng = np.random.default_rng(0)
    y = rng.standard_normal(geo.M) + 1j * rng.standard_normal(geo.M)
    s = np.zeros(geo.N, dtype=np.complex128)
    seq = np.random.default_rng(configs.SEEDS["minibatch"])
    times = []
    while len(times) < w.iters and (sum(times) < budget_s or len(times) < 3):
        idx = np.sort(seq.choice(geo.M, w.batch, replace=False))
        t1 = time.perf_counter()
        g = op.adjoint(op.forward(s, idx, threads) - y[idx], idx, threads) / idx.size
        s = O.soft_threshold(s - 1e-3 * g, 1e-6)
        times.append(time.perf_counter() - t1)
    per = float(np.mean(times[1:]))
    print(json.dumps({
        "workload": workload, "value": 2.0 * w.batch * geo.N / per, "unit": UNIT, "iters_per_s": 1.0 / per,
        "s_per_iter": per, "iters_timed": len(times), "iters_of_config": w.iters, "cores": threads, "kind": "port",
        "plan_build_s": build_s, "table_bytes": O.TableOperator.table_bytes(geo),
        "peak_rss_bytes": _vm_hwm_bytes(), "rss_before_tables_bytes": rss0, "rss_after_tables_bytes": rss_tables,
        "sample": f"full {workload} grid (N={geo.N}, M={geo.M}), |B|={w.batch} flat, the oracle's table restatement "
                  f"of the reference algorithm (forward.py:183-336, solver.py:181-241); plan build and peak RSS "
                  f"reported separately (BASELINE.md §3)",
    }), flush=True)
    return 0


def hbm_peak_gbs() -> float:
    try:
        return float(json.load(open(ROOT / "MEASURED_PEAKS.json"))["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback (6.65 TB/s copy bandwidth)


def ncu_traffic(kernel: str):
    """dram read+write bytes per launch of the dominant kernel from the committed ncu --set full
    capture (profiles/*_ncu_summary.json; ncu's numbers, not measured by this run), or None."""
    files = sorted((ROOT / "profiles").glob("r*_ncu_summary.json"))
    if not files:
        return None
    try:
        d = json.load(open(files[-1]))
        key = next(k for k in d if k.startswith("fwd_kernel" if kernel == "forward" else "adj_kernel<float, 1"))
        b = d[key]["dram__bytes_read.sum"] + d[key]["dram__bytes_write.sum"]  # base units (bytes)
        return {"bytes_per_launch": b, "source": files[-1].name, "unit": "B"}
    except Exception:
        return None


def kernel_times(eng, plan, seed, k0, reps):
    import torch

    st = torch.cuda.current_stream()
    B = plan.B
    f_ms, a_ms = [], []
    for i in range(reps):
        eng.sample_device(seed, k0 + i, B)
        yb = eng.ybuf[:B]
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        c = torch.cuda.Event(enable_timing=True)
        a.record(st)
        if eng.collective == "peer":
            plan.forward_allreduce(eng.s, out=yb)
        else:
            plan.forward(eng.s, out=yb)
        b.record(st)
        if eng.pg is not None and eng.collective != "peer":
            torch.distributed.all_reduce(torch.view_as_real(yb), group=eng.pg)
        c0 = torch.cuda.Event(enable_timing=True)
        c0.record(st)
        plan.adjoint_prox(yb, eng.y, eng.s, eng.s_next, eng.eta / B, eng.alpha, eng.stats)
        c.record(st)
        eng.s, eng.s_next = eng.s_next, eng.s
        torch.cuda.synchronize()
        f_ms.append(a.elapsed_time(b))
        a_ms.append(c0.elapsed_time(c))
    return {"fwd_ms": float(np.median(f_ms)), "adj_ms": float(np.median(a_ms))}


def e2e_public_api(w, eng, args):
    """End to end through the reference's own entry point, spgm_solve (solver.py:349), as a user calls it:
    numpy y on the host, flat minibatches drawn on the host with the reference's numpy call sequence
    (sorted choice without replacement from one persistent generator), each iteration's index list copied
    H2D, each iteration's termination statistics copied D2H and checked (reference semantics: a record per
    iteration, tolerance test every iteration), the final volume copied back. The plan is built by a short
    warm-up call (plan cache) outside the timed region; everything else is inside it."""
    from paper_2509_00774_b200.solver import SolverConfig, spgm_solve

    scn = w.scenario
    y = eng.y.to(torch_complex128()).cpu().numpy()
    iters = max(args.steps, 100)

    def cfg(n):
        return SolverConfig(eta=eng.eta, alpha=eng.alpha, max_iters=n, tol=1e-300, dtype=w.dtype,
                            flat_batch=w.batch, sampler="host", rng_seed=1234)

    spgm_solve(y, scn, cfg(3))  # warm: plan cache, kernel attributes
    t0 = time.perf_counter()
    rep = spgm_solve(y, scn, cfg(iters))
    dt = time.perf_counter() - t0
    assert rep.iterations == iters and len(rep.per_iteration) == iters
    return {"value": 2.0 * w.batch * scn.n_voxels * iters / dt, "unit": UNIT, "h2d_bytes_per_step": 4 * w.batch,
            "d2h_bytes_per_step": 32, "ms_per_step": dt / iters * 1e3, "iterations": iters,
            "how": "wall clock around paper_2509_00774_b200.spgm_solve (the reference's entry point, solver.py:349) "
                   "for the full solve: host numpy flat sampling as the reference, H2D of each iteration's "
                   "indices, D2H + tolerance check of each iteration's statistics, one IterationRecord per "
                   "iteration, the final volume D2H (plus y H2D once per solve)"}


def torch_complex128():
    import torch

    return torch.complex128


def e2e_run(eng, scn, B, N, args, pg, local):
    """End to end through the public engine: per step, the host draws the flat minibatch with numpy
    (sorted choice without replacement, as the reference's sampler does on the CPU), uploads it from
    pinned memory, runs the step, and reads the step's termination statistics back. The loop is
    pipelined like a production driver: the host draws batch k+1 and reads step k's statistics
    (one async D2H per step into a pinned double buffer) while the GPU runs step k+1."""
    import torch
    import torch.distributed as dist

    rng = np.random.default_rng(1234)
    M = scn.n_channels
    steps = args.steps
    dev = eng.plan.device
    bufs = [torch.empty(B, dtype=torch.int32).pin_memory() for _ in range(2)]
    stats_host = torch.empty((2, 4), dtype=torch.float64).pin_memory()
    events = [torch.cuda.Event() for _ in range(2)]
    st = torch.cuda.current_stream()
    changes = []

    def draw(k):
        bufs[k % 2].copy_(torch.from_numpy(np.sort(rng.choice(M, B, replace=False)).astype(np.int32)))

    def launch(k):
        eng.idx_dev[:B].copy_(bufs[k % 2], non_blocking=True)  # H2D of this step's indices
        eng.plan.prepare(eng.idx_dev[:B])
        eng.step_staged()
        stats = eng.stats
        if pg is not None:
            stats = stats.clone()
            dist.all_reduce(stats, group=pg)
        stats_host[k % 2].copy_(stats, non_blocking=True)  # D2H of this step's result
        events[k % 2].record(st)

    def consume(k):
        events[k % 2].synchronize()
        s0, s1 = float(stats_host[k % 2, 0]), float(stats_host[k % 2, 1])
        changes.append(s1 ** 0.5 / max(s0 ** 0.5, 1e-300))

    for k in range(2):  # warm-up
        draw(k)
        launch(k)
        consume(k)
    if pg is not None:
        dist.barrier(device_ids=[local])
    torch.cuda.synchronize(dev)
    changes.clear()
    t0 = time.perf_counter()
    draw(0)
    for k in range(steps):
        launch(k)
        if k + 1 < steps:
            draw(k + 1)  # host work overlaps step k on the GPU
        if k > 0:
            consume(k - 1)
    consume(steps - 1)
    torch.cuda.synchronize(dev)
    dt = time.perf_counter() - t0
    if pg is not None:
        t = torch.tensor([dt], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    assert len(changes) == steps
    return {"value": 2.0 * B * N * steps / dt, "unit": UNIT, "h2d_bytes_per_step": 4 * B,
            "d2h_bytes_per_step": 32, "ms_per_step": dt / steps * 1e3,
            "how": "wall clock around spgm steps: host numpy flat sampling (sorted choice without replacement, "
                   "as the reference), pinned H2D of each step's index list, D2H of each step's termination "
                   "stats; the host samples step k+1 and reads step k's stats while the GPU runs step k+1"}


def main():
    args = parse()
    if args.cpu_child:
        return cpu_child_main(args.cpu_child, args.cpu_seconds)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
