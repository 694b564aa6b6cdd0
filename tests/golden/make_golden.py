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
        pulse=_ref_pulse(scn.pulse),
        c=scn.c,
    )


def _ref_pulse(p):
    if hasattr(p, "frequencies_hz"):
        return ref.TabulatedPulse(tuple(p.frequencies_hz), tuple(p.values))
    return ref.ConstantPulse(p.value)


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


def gen_baseline_medium():
    """BASELINE config 1 ('Medium') end to end with the reference's operator: scene, noise, L (20 power
    iterations), lambda, and the 300-iteration flat SPGM loop through ref.minibatch_gradient and
    ref.soft_threshold (solver.py:181-183, 228-241), the index table drawn as the reference's
    sampler would (one default_rng(0) across iterations). The reference run holds the 4.3 GB tables."""
    w = configs.WORKLOADS["medium"]()
    scn = to_ref(w.scenario)
    threads = os.cpu_count() or 1
    t0 = time.time()
    s_true = configs.make_scene(w)
    clean = ref.forward_apply(s_true, scn, threads=threads)
    sigma = configs.noise_sigma(clean, w.snr_db)
    y = ref.simulate_measurements(s_true, scn, noise_sigma=sigma, rng_seed=configs.SEEDS["noise"],
                                  threads=threads).values
    L = ref.lipschitz_estimate(scn, n_iters=20, rng_seed=configs.SEEDS["power"], threads=threads)
    M = scn.n_channels
    lam = 1e-3 * float(np.max(np.abs(ref.adjoint_apply(y, scn, threads=threads)))) / M
    eta = 1.0 / L
    alpha = eta * lam
    print(f"medium setup: {time.time() - t0:.1f}s  L={L:.6e}")
    rng = np.random.default_rng(configs.SEEDS["minibatch"])
    table = np.stack([np.sort(rng.choice(M, w.batch, replace=False)) for _ in range(w.iters)])
    s = np.zeros(scn.n_voxels, dtype=np.complex128)
    changes = []
    for idx in table:
        g = ref.minibatch_gradient(s, y, scn, idx, threads=threads)
        s_next = ref.soft_threshold(s - eta * g, alpha)
        changes.append(ref.relative_magnitude_change(s, s_next))
        s = s_next
    print(f"medium 300 iterations done: {time.time() - t0:.1f}s")
    np.savez_compressed(
        OUT / "baseline_medium.npz",
        fingerprint=np.frombuffer(ref.scenario_fingerprint(scn), dtype=np.uint8),
        sigma=np.array(sigma), y=y, L=np.array(L), lam=np.array(lam), eta=np.array(eta), alpha=np.array(alpha),
        index_table=table.astype(np.int32), s_final=s, changes=np.array(changes),
    )


def _sparse(v):
    nz = np.flatnonzero(v)
    return nz.astype(np.int32), v[nz]


def gen_paper_v():
    """The paper-v study of the reference's acceptance suite (test_acceptance.py:69-106, 201-308) run
    by the reference itself: the converged PGM reconstruction at 30 dB, three seeded SPGM(4,4,3) runs
    and their PSNR against it (criterion 6), and the single-scatterer localisation (criterion 9).
    Volumes are stored sparse (the l1 prox zeroes most voxels)."""
    paper = ref.preset_scenario("paper-v")
    out = {"fingerprint": np.frombuffer(ref.scenario_fingerprint(paper), dtype=np.uint8)}
    t0 = time.time()
    phantom = ref.make_phantom("points:5", paper.voxels, rng_seed=42)
    clean = ref.forward_apply(phantom, paper)
    sigma = float(np.sqrt(np.mean(np.abs(clean) ** 2) * 10 ** (-30 / 10)))
    y = ref.simulate_measurements(phantom, paper, noise_sigma=sigma, rng_seed=7).values
    out["y"] = y
    out["sigma"] = np.array(sigma)
    pgm = ref.pgm_solve(y, paper, ref.SolverConfig(eta=1e-3, alpha=4e-5, tol=1e-3, max_iters=2000))
    print(f"paper-v PGM: {pgm.iterations} iterations, {pgm.termination}, {time.time() - t0:.1f}s")
    out["pgm_iterations"] = np.array(pgm.iterations)
    out["pgm_changes"] = np.array([r.magnitude_change for r in pgm.per_iteration])
    out["pgm_nz"], out["pgm_val"] = _sparse(pgm.volume.values)
    for seed in (1, 2, 3):
        rep = ref.spgm_solve(y, paper, ref.SolverConfig(eta=1e-3, alpha=4e-5, tol=1e-3, max_iters=4000,
                                                        composition=ref.MinibatchComposition(4, 4, 3),
                                                        rng_seed=seed))
        psnr = ref.psnr_vs_reference(rep.volume, pgm.volume).psnr_db
        print(f"paper-v SPGM seed {seed}: {rep.iterations} iterations, PSNR {psnr:.3f} dB, {time.time() - t0:.1f}s")
        out[f"spgm{seed}_iterations"] = np.array(rep.iterations)
        out[f"spgm{seed}_psnr"] = np.array(psnr)
        out[f"spgm{seed}_changes"] = np.array([r.magnitude_change for r in rep.per_iteration])
        out[f"spgm{seed}_nz"], out[f"spgm{seed}_val"] = _sparse(rep.volume.values)
    truth = ref.make_phantom("points:1", paper.voxels, rng_seed=13)
    y1 = ref.simulate_measurements(truth, paper, noise_sigma=0.0).values
    rep = ref.pgm_solve(y1, paper, ref.SolverConfig(eta=1e-3, alpha=4e-5, tol=1e-3, max_iters=150))
    out["loc_true_voxel"] = np.array(int(np.argmax(np.abs(truth.values))))
    out["loc_found_voxel"] = np.array(int(np.argmax(np.abs(rep.volume.values))))
    out["loc_iterations"] = np.array(rep.iterations)
    out["loc_nz"], out["loc_val"] = _sparse(rep.volume.values)
    print(f"paper-v localisation: {int(out['loc_found_voxel'])} vs {int(out['loc_true_voxel'])}, "
          f"{time.time() - t0:.1f}s")
    np.savez_compressed(OUT / "paper_v_study.npz", **out)


def gen_pulse():
    """Frequency-dependent complex pulse (TabulatedPulse, geometry.py:239-269) through the reference's
    forward (p_f, forward.py:283-284), adjoint (conj p_f, :315-325) and a structured SPGM run."""
    sys.path.insert(0, str(ROOT / "tests"))
    import pulse_cases

    out = {}
    for name, build in pulse_cases.CASES.items():
        scn = to_ref(build())
        M, N = scn.n_channels, scn.n_voxels
        rng = np.random.default_rng(31)
        s = rc(rng, N)
        threads = os.cpu_count() or 1
        out[f"{name}_fingerprint"] = np.frombuffer(ref.scenario_fingerprint(scn), dtype=np.uint8)
        if name != "medium":  # Medium's s is regenerated from default_rng(31) by the test (2 MB)
            out[f"{name}_s"] = s
        if name == "medium":
            idx = np.sort(rng.choice(M, 512, replace=False))
            r = rc(rng, idx.size)
            out["medium_idx"] = idx.astype(np.int32)
            out["medium_r"] = r
            out["medium_fwd_sub"] = ref.forward_apply(s, scn, subset=idx, threads=threads)
            adj = ref.adjoint_apply(r, scn, subset=idx, threads=threads)
            probe = np.sort(rng.choice(N, 4096, replace=False))
            out["medium_adj_probe_voxels"] = probe.astype(np.int64)
            out["medium_adj_sub_probe"] = adj[probe]
            continue
        r = rc(rng, M)
        sub = np.sort(rng.choice(M, max(1, M // 3), replace=False))
        out[f"{name}_r"] = r
        out[f"{name}_sub"] = sub
        out[f"{name}_fwd"] = ref.forward_apply(s, scn)
        out[f"{name}_fwd_sub"] = ref.forward_apply(s, scn, subset=sub)
        out[f"{name}_adj"] = ref.adjoint_apply(r, scn)
        out[f"{name}_adj_sub"] = ref.adjoint_apply(r[: sub.size], scn, subset=sub)
        y = rc(np.random.default_rng(32), M)
        out[f"{name}_y"] = y
        T, R, F = scn.array.n_tx, scn.array.n_rx, scn.frequencies.count
        comp = ref.MinibatchComposition(max(1, F // 2), max(1, T - 1), max(1, R - 1))
        out[f"{name}_comp"] = np.array([comp.n_f, comp.n_tx, comp.n_rx])
        eta = 0.9 / ref.lipschitz_estimate(scn, n_iters=200, tol=1e-12)
        alpha = 0.05 * eta * float(np.max(np.abs(ref.adjoint_apply(y, scn)))) / M
        out[f"{name}_eta_alpha"] = np.array([eta, alpha])
        rep = ref.spgm_solve(y, scn, ref.SolverConfig(eta=eta, alpha=alpha, max_iters=10, tol=1e-300,
                                                      composition=comp, rng_seed=4))
        out[f"{name}_spgm"] = rep.volume.values
    np.savez_compressed(OUT / "pulse_scenarios.npz", **out)


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
    if "medium_spgm" in which:
        gen_baseline_medium()
    if "paper_v" in which:
        gen_paper_v()
    if "pulse" in which:
        gen_pulse()
    print("fixtures written to", OUT)
