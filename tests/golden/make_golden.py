#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ from the REFERENCE implementation.

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py

It imports the unmodified reference package ``nfmimo`` (pkg/src/nfmimo) and records
its outputs on seeded inputs. The GPU box has no /root/reference, so the tests
compare against these committed arrays. Scenarios are rebuilt from plain
parameters on both sides, and each fixture also records the reference's scenario
fingerprint. That pins the product's geometry restatement too.
"""

from __future__ import annotations

import math
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

REF = os.environ.get("NFMIMO_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
import nfmimo as ref  # noqa: E402

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2509_00774_b200 import configs  # noqa: E402  (scenario parameters only)

OUT = Path(__file__).resolve().parent


def to_ref(scn) -> "ref.ImagingScenario":
    """Rebuild a product ImagingScenario with the reference's own types."""
    a = scn.array
    return ref.ImagingScenario(
        array=ref.ArrayGeometry(
            tuple(ref.Vec3(p.x, p.y, p.z) for p in a.transmitters),
            tuple(ref.Vec3(p.x, p.y, p.z) for p in a.receivers),
        ),
        frequencies=ref.FrequencyGrid(scn.frequencies.f_start, scn.frequencies.f_stop, scn.frequencies.count),
        voxels=ref.VoxelGrid(
            center=ref.Vec3(scn.voxels.center.x, scn.voxels.center.y, scn.voxels.center.z),
            extent=scn.voxels.extent,
            dims=scn.voxels.dims,
        ),
        pulse=ref.ConstantPulse(scn.pulse.value),
        c=scn.c,
    )


def rc(rng, n):
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


def tiny_ref():
    return ref.ImagingScenario(
        array=ref.ArrayGeometry(
            transmitters=(ref.Vec3(0.05, 0.0, 0.0), ref.Vec3(-0.05, 0.02, 0.0)),
            receivers=(ref.Vec3(0.0, 0.04, 0.0), ref.Vec3(0.01, -0.03, 0.0)),
        ),
        frequencies=ref.FrequencyGrid(5e9, 7e9, 2),
        voxels=ref.VoxelGrid(center=ref.Vec3(0.0, 0.0, 0.35), extent=(0.1, 0.1, 0.0), dims=(2, 2, 1)),
    )


def small_ref():
    return ref.ImagingScenario(
        array=ref.make_spiral_array(3, 2, 0.15, rng_seed=3),
        frequencies=ref.FrequencyGrid(4e9, 9e9, 3),
        voxels=ref.VoxelGrid(center=ref.Vec3(0.0, 0.0, 0.3), extent=(0.12, 0.08, 0.06), dims=(3, 2, 2)),
    )


def gen_unit_scenarios():
    """Dense matrices and operator outputs of the reference tests' fixture scenarios."""
    out = {}
    for name, scn in (("tiny", tiny_ref()), ("small", small_ref())):
        rng = np.random.default_rng(2024)
        dense = ref.materialize_dense(scn)
        s = rc(rng, scn.n_voxels)
        r = rc(rng, scn.n_channels)
        sub = rng.choice(scn.n_channels, size=max(1, scn.n_channels // 2), replace=False)
        out[f"{name}_fingerprint"] = np.frombuffer(ref.scenario_fingerprint(scn), dtype=np.uint8)
        out[f"{name}_dense"] = dense
        out[f"{name}_s"] = s
        out[f"{name}_r"] = r
        out[f"{name}_sub"] = sub
        out[f"{name}_fwd"] = ref.forward_apply(s, scn)
        out[f"{name}_fwd_sub"] = ref.forward_apply(s, scn, subset=sub)
        out[f"{name}_adj"] = ref.adjoint_apply(r, scn)
        out[f"{name}_adj_sub"] = ref.adjoint_apply(r[: sub.size], scn, subset=sub)
    scn = small_ref()
    out["small_lipschitz"] = np.array(ref.lipschitz_estimate(scn, n_iters=500, tol=1e-13))
    rng = np.random.default_rng(12345)
    y = rc(rng, scn.n_channels)
    out["small_y"] = y
    comp = ref.MinibatchComposition(2, 2, 1)
    rep = ref.spgm_solve(y, scn, ref.SolverConfig(max_iters=30, tol=1e-300, composition=comp, rng_seed=9))
    out["small_spgm_structured"] = rep.volume.values
    out["small_spgm_changes"] = np.array([r.magnitude_change for r in rep.per_iteration])
    rep = ref.pgm_solve(y, scn, ref.SolverConfig(max_iters=25, tol=1e-300))
    out["small_pgm"] = rep.volume.values
    idx_seq = [ref.sample_minibatch(comp, scn, np.random.default_rng(9)).indices]
    out["small_structured_first_batch"] = idx_seq[0]
    np.savez_compressed(OUT / "unit_scenarios.npz", **out)


def gen_baseline_small():
    """BASELINE config 0 ('Small', c128) end to end with the reference's operator."""
    w = configs.WORKLOADS["small"]()
    scn = to_ref(w.scenario)
    s_true = configs.make_scene(w)
    clean = ref.forward_apply(s_true, scn)
    sigma = configs.noise_sigma(clean, w.snr_db)
    y = ref.simulate_measurements(s_true, scn, noise_sigma=sigma, rng_seed=configs.SEEDS["noise"]).values
    L = ref.lipschitz_estimate(scn, n_iters=20, rng_seed=configs.SEEDS["power"])
    M = scn.n_channels
    lam = 1e-3 * float(np.max(np.abs(ref.adjoint_apply(y, scn)))) / M
    eta = 1.0 / L
    alpha = eta * lam
    rng = np.random.default_rng(configs.SEEDS["minibatch"])
    table = np.stack([np.sort(rng.choice(M, w.batch, replace=False)) for _ in range(w.iters)])
    s = np.zeros(scn.n_voxels, dtype=np.complex128)
    changes = []
    snapshots = {}
    for k, idx in enumerate(table, start=1):
        g = ref.minibatch_gradient(s, y, scn, idx)
        s_next = ref.soft_threshold(s - eta * g, alpha)
        changes.append(ref.relative_magnitude_change(s, s_next))
        s = s_next
        if k in (1, 10, 50):
            snapshots[f"s_iter{k}"] = s.copy()
    rng = np.random.default_rng(77)
    probe_s = rc(rng, scn.n_voxels)
    probe_r = rc(rng, w.batch)
    np.savez_compressed(
        OUT / "baseline_small.npz",
        fingerprint=np.frombuffer(ref.scenario_fingerprint(scn), dtype=np.uint8),
        s_true=s_true, clean=clean, sigma=np.array(sigma), y=y, L=np.array(L), lam=np.array(lam),
        eta=np.array(eta), alpha=np.array(alpha), index_table=table.astype(np.int32),
        s_final=s, changes=np.array(changes),
        probe_s=probe_s, probe_r=probe_r, probe_idx=table[0],
        probe_fwd=ref.forward_apply(probe_s, scn, subset=table[0]),
        probe_adj=ref.adjoint_apply(probe_r, scn, subset=table[0]),
        **snapshots,
    )


def gen_medium_ops():
    """BASELINE config 1 ('Medium') operator outputs from the reference (4.3 GB of tables)."""
    w = configs.WORKLOADS["medium"]()
    scn = to_ref(w.scenario)
    M, N = scn.n_channels, scn.n_voxels
    rng = np.random.default_rng(123)
    s = rc(rng, N)
    idx = np.sort(np.random.default_rng(configs.SEEDS["minibatch"]).choice(M, w.batch, replace=False))
    r = rc(np.random.default_rng(124), w.batch)
    t0 = time.time()
    fwd = ref.forward_apply(s, scn, subset=idx, threads=8)
    adj = ref.adjoint_apply(r, scn, subset=idx, threads=8)
    print(f"medium reference ops: {time.time() - t0:.1f}s")
    probe = np.sort(np.random.default_rng(125).choice(N, 8192, replace=False))
    np.savez_compressed(
        OUT / "medium_ops.npz",
        fingerprint=np.frombuffer(ref.scenario_fingerprint(scn), dtype=np.uint8),
        s_seed=np.array(123), r_seed=np.array(124), idx=idx.astype(np.int32), fwd=fwd,
        adj_probe_voxels=probe.astype(np.int64), adj_probe=adj[probe], adj_norm=np.array(np.linalg.norm(adj)),
    )


def gen_known_answers():
    """The reference tests' scalar known answers, evaluated by the reference itself."""
    c = ref.SPEED_OF_LIGHT

    def one(tx, rx, vox, f):
        return ref.ImagingScenario(
            array=ref.ArrayGeometry((ref.Vec3(*tx),), (ref.Vec3(*rx),)),
            frequencies=ref.FrequencyGrid(f, f, 1),
            voxels=ref.VoxelGrid(center=ref.Vec3(*vox), extent=(0, 0, 0), dims=(1, 1, 1)),
        )

    golden = ref.matrix_element(0, 0, one((0.1, 0, 0), (-0.1, 0, 0), (0, 0, 0.4), 10e9))
    full = ref.matrix_element(0, 0, one((0, 0, 0), (0, 0, 0), (0, 0, 0.5), c))
    quarter = ref.matrix_element(0, 0, one((0, 0, 0), (0, 0, 0), (0, 0, 0.5), c / 4))
    np.savez_compressed(
        OUT / "known_answers.npz",
        golden_element=np.array(golden), full_wave=np.array(full), quarter_wave=np.array(quarter),
        soft_in=np.array([3 + 4j]), soft_alpha=np.array(2.0), soft_out=ref.soft_threshold(np.array([3 + 4j]), 2.0),
        change=np.array(ref.relative_magnitude_change(np.array([1.0 + 0j, 0.0]), np.array([1.1 + 0j, 0.0]))),
    )


if __name__ == "__main__":
    which = sys.argv[1:] or ["known", "unit", "small", "medium"]
    if "known" in which:
        gen_known_answers()
    if "unit" in which:
        gen_unit_scenarios()
    if "small" in which:
        gen_baseline_small()
    if "medium" in which:
        gen_medium_ops()
    print("fixtures written to", OUT)
