"""The persistent SPGM loop (nf_spgm_loop, spgm_loop_kernel): K iterations of solver._solve
(solver.py:259-318) per cooperative launch, with the batch sort, forward, reduce, residual, adjoint +
prox and termination statistics between grid barriers. It runs the same arithmetic in the same order
as the per-launch path, so its iterates must equal nf_batch_prepare + nf_forward + nf_adjoint_prox
bit for bit, and spgm_solve / pgm_solve must return the same report either way (NFGPU_LOOP=0 forces
the per-iteration path)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden, rc, rel_l2
from paper_2509_00774_b200 import MinibatchComposition, SolverConfig, configs, pgm_solve, spgm_solve
from paper_2509_00774_b200.plan import DevicePlan
from paper_2509_00774_b200.solver import SPGMEngine

pytestmark = pytest.mark.gpu


@pytest.fixture
def no_tiny(monkeypatch):
    """Keep small problems on spgm_loop_kernel (the flat kernels' arithmetic) instead of tiny_loop_kernel."""
    monkeypatch.setenv("NFGPU_TINY", "0")


def _pair(scn, dtype, y, eta, alpha, s0=None, max_batch=None):
    engs = []
    for _ in range(2):
        plan = DevicePlan(scn, dtype=dtype, device="cuda:0", max_batch=max_batch, structured="never")
        engs.append(SPGMEngine(plan, y, eta, alpha, initial=s0))
    return engs


@pytest.mark.parametrize("ct", ["auto", "forced", "forward-only", "equal-ranges"])
@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("workload", ["small", "medium"])
def test_loop_matches_per_launch_path_bitwise(workload, dtype, ct, no_tiny, monkeypatch):
    """ct="forced" (NFGPU_CT=2) runs the CTA-tile forward and adjoint wherever their layout fits, Small included,
    in both paths."""
    if ct == "forced":
        monkeypatch.setenv("NFGPU_CT", "2")
    elif ct == "forward-only":  # CTA-tile forward beside the warp-unit adjoint
        monkeypatch.setenv("NFGPU_CT", "2")
        monkeypatch.setenv("NFGPU_CT_ADJ", "0")
    elif ct == "equal-ranges":  # no cost-balanced cuts (ct_args)
        monkeypatch.setenv("NFGPU_CT", "2")
        monkeypatch.setenv("NFGPU_CT_COST_FWD", "0")
        monkeypatch.setenv("NFGPU_CT_COST_ADJ", "0")
    w = configs.WORKLOADS[workload]()
    scn = w.scenario
    rng = np.random.default_rng(3)
    y = rc(rng, scn.n_channels)
    s0 = rc(rng, scn.n_voxels) * 0.01
    eta, alpha = 1e-3, 1e-7
    a, b = _pair(scn, dtype, y, eta, alpha, s0, max_batch=w.batch)
    K = 9
    table = np.stack([np.sort(rng.choice(scn.n_channels, w.batch, replace=False)) for _ in range(K)])
    stats = []
    for k in range(K):
        a.stage(table[k])
        a.step_staged()
        stats.append(a.stats.clone())
    b.run_loop(K, table=table, tol=0.0)
    n, reason = b.loop_result()
    assert (n, reason) == (K, 0)
    assert torch.equal(a.s, b.s)
    rec = b._loop_rec[:K, :4]
    assert torch.equal(torch.stack(stats), rec)


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_loop_many_tiles_large_batch_bitwise(dtype):
    """2048 tiles and |B| = 4096: a CTA's partials [tiles][28 channels] do not fit in shared memory at once, so the
    loop's reduce phase stages them in chunks of tiles and keeps its running segment sums between chunks; the
    iterates must still equal the per-launch path's bit for bit."""
    from paper_2509_00774_b200 import ArrayGeometry, FrequencyGrid, ImagingScenario, Vec3, VoxelGrid

    rng = np.random.default_rng(9)
    tx = rng.uniform(-0.1, 0.1, size=(4, 2))
    rx = rng.uniform(-0.1, 0.1, size=(4, 2))
    scn = ImagingScenario(
        array=ArrayGeometry(tuple(Vec3(a, b, 0.0) for a, b in tx), tuple(Vec3(a, b, 0.0) for a, b in rx)),
        frequencies=FrequencyGrid(57e9, 64e9, 512),
        voxels=VoxelGrid(center=Vec3(0.0, 0.0, 0.4), extent=(0.3, 0.3, 0.2), dims=(128, 64, 64)),
    )
    B, K = 4096, 3
    y = rc(rng, scn.n_channels)
    s0 = rc(rng, scn.n_voxels) * 0.01
    a, b = _pair(scn, dtype, y, 1e-3, 1e-7, s0, max_batch=B)
    table = np.stack([np.sort(rng.choice(scn.n_channels, B, replace=False)) for _ in range(K)])
    stats = []
    for k in range(K):
        a.stage(table[k])
        a.step_staged()
        stats.append(a.stats.clone())
    b.run_loop(K, table=table, tol=0.0)
    assert b.loop_result() == (K, 0)
    assert torch.equal(a.s, b.s)
    assert torch.equal(torch.stack(stats), b._loop_rec[:K, :4])


@pytest.mark.parametrize("dtype", ["c128", "c64"])
def test_loop_device_sampler_matches_per_launch(dtype, no_tiny):
    w = configs.WORKLOADS["small"]()
    scn = w.scenario
    rng = np.random.default_rng(4)
    y = rc(rng, scn.n_channels)
    a, b = _pair(scn, dtype, y, 2e-3, 1e-6, max_batch=w.batch)
    for k in range(1, 8):
        a.sample_device(11, k, w.batch)
        a.step_staged()
    b.run_loop(7, table=None, seed=11, iter0=1, batch=w.batch, tol=0.0)
    assert b.loop_result() == (7, 0)
    assert torch.equal(a.s, b.s)


@pytest.mark.parametrize("dtype,tol", [("c128", 1e-10), ("c64", 1e-4)])
def test_baseline_small_through_the_loop(dtype, tol):
    """BASELINE config 0 end to end on the persistent loop (host flat sampler, reference call sequence):
    the reference's 200-iteration reconstruction, and the same report as the per-iteration path."""
    b = golden("baseline_small")
    scn = configs.small_scenario()
    cfg = SolverConfig(eta=float(b["eta"]), alpha=float(b["alpha"]), max_iters=200, tol=1e-300, dtype=dtype,
                       flat_batch=32, rng_seed=0)
    rep = spgm_solve(b["y"], scn, cfg)
    assert rep.iterations == 200 and rep.termination == "max_iters"
    assert rel_l2(rep.volume.values, b["s_final"]) <= tol
    changes = np.array([r.magnitude_change for r in rep.per_iteration])
    assert np.allclose(changes, b["changes"], rtol=1e-6 if dtype == "c128" else 2e-2)
    assert all(r.elapsed_seconds > 0 for r in rep.per_iteration)
    import os

    os.environ["NFGPU_LOOP"] = "0"
    try:
        rep0 = spgm_solve(b["y"], scn, cfg)
    finally:
        os.environ.pop("NFGPU_LOOP")
    # Small runs on tiny_loop_kernel (entries from the geometry in fp64, its own summation order): the same
    # reconstruction as the per-iteration flat kernels to the dtype's tolerance
    assert rel_l2(rep.volume.values, rep0.volume.values) <= (1e-11 if dtype == "c128" else 1e-5)


def test_loop_terminations_match_per_iteration_path(monkeypatch, no_tiny):
    """Tolerance stop mid-chunk and across chunk boundaries (LOOP_CHUNK), the full-batch PGM path on a
    flat-routed scenario, the table and composition samplers, and the time budget."""
    from paper_2509_00774_b200 import solver as S

    scn = configs.small_scenario()
    rng = np.random.default_rng(5)
    s_true = np.zeros(scn.n_voxels, complex)
    s_true[rng.choice(scn.n_voxels, 5, replace=False)] = 1.0
    from paper_2509_00774_b200 import forward_apply, lipschitz_estimate

    y = forward_apply(s_true, scn)
    eta = 0.9 / lipschitz_estimate(scn, n_iters=50)
    monkeypatch.setattr(S, "LOOP_CHUNK", 7)

    def both(fn, cfg):
        r1 = fn(y, scn, cfg)
        monkeypatch.setenv("NFGPU_LOOP", "0")
        r0 = fn(y, scn, cfg)
        monkeypatch.delenv("NFGPU_LOOP")
        return r1, r0

    for cfg, fn in [
        (SolverConfig(eta=eta, alpha=1e-6, tol=2e-3, max_iters=500, flat_batch=64, rng_seed=1), spgm_solve),
        (SolverConfig(eta=eta, alpha=1e-6, tol=1e-3, max_iters=300), pgm_solve),
        (SolverConfig(eta=eta, alpha=1e-6, tol=1e-300, max_iters=23, composition=MinibatchComposition(3, 2, 2),
                      rng_seed=2), spgm_solve),
        (SolverConfig(eta=eta, alpha=1e-6, tol=1e-300, max_iters=15, sampler="table",
                      index_table=np.stack([np.sort(rng.choice(scn.n_channels, 40, replace=False))
                                            for _ in range(15)])), spgm_solve),
        (SolverConfig(eta=eta, alpha=1e-6, tol=1e-300, max_iters=20, flat_batch=16, sampler="device",
                      rng_seed=9), spgm_solve),
    ]:
        r1, r0 = both(fn, cfg)
        assert r1.iterations == r0.iterations and r1.termination == r0.termination
        assert np.array_equal(r1.volume.values, r0.volume.values)
        assert [r.magnitude_change for r in r1.per_iteration] == [r.magnitude_change for r in r0.per_iteration]
        assert [r.batch_size for r in r1.per_iteration] == [r.batch_size for r in r0.per_iteration]
    # time budget: stops early on the device clock
    rep = spgm_solve(y, scn, SolverConfig(eta=eta, alpha=1e-6, tol=1e-300, max_iters=10_000_000, flat_batch=32,
                                          time_budget_s=0.05))
    assert rep.termination == "time_budget" and 1 <= rep.iterations < 10_000_000
    assert len(rep.per_iteration) == rep.iterations


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("dims", [(16, 16, 8), (13, 6, 5), (3, 2, 1)])
def test_tiny_loop_step_matches_oracle(dims, dtype):
    """tiny_loop_kernel (|B|·N <= 2^20): one SPGM step against the oracle's direct formula, on the BASELINE Small
    array with grids that do and do not fill its 256-voxel blocks, with a tabulated complex pulse."""
    import pulse_cases
    from oracle import nfmimo_oracle as O
    from paper_2509_00774_b200 import ImagingScenario, Vec3, VoxelGrid

    base = configs.small_scenario()
    scn = ImagingScenario(array=base.array, frequencies=base.frequencies,
                          voxels=VoxelGrid(center=Vec3(0, 0, 0.3),
                                           extent=tuple(0.0 if d == 1 else e for d, e in zip(dims, (0.2, 0.2, 0.1))),
                                           dims=dims),
                          pulse=pulse_cases.tabulated_pulse(60e9, 64e9, seed=5), c=base.c)
    geo = O.geom_from_scenario(scn)
    rng = np.random.default_rng(8)
    s, y = rc(rng, scn.n_voxels), rc(rng, scn.n_channels)
    idx = np.sort(rng.choice(scn.n_channels, 32, replace=False))
    grad = O.direct_adjoint(geo, O.direct_forward(geo, s, idx) - y[idx], idx) / idx.size
    eta = 0.5 / float(np.max(np.abs(grad)))
    alpha = 0.3 * float(np.median(np.abs(s - eta * grad)))
    ref = O.soft_threshold(s - eta * grad, alpha)
    plan = DevicePlan(scn, dtype=dtype, device="cuda:0", max_batch=32)
    eng = SPGMEngine(plan, y, eta, alpha, initial=s)
    eng.run_loop(1, table=idx[None, :], tol=0.0)
    assert eng.loop_result() == (1, 0)
    assert rel_l2(eng.volume(), ref) <= (1e-10 if dtype == "c128" else 1e-5)
    rec = eng._loop_rec[0].cpu().numpy()
    assert rec[2] == pytest.approx(0.5 * np.sum(np.abs(O.direct_forward(geo, s, idx) - y[idx]) ** 2), rel=1e-6)
    change = np.sqrt(rec[1]) / np.sqrt(rec[0])
    assert change == pytest.approx(O.relative_magnitude_change(s, ref), rel=1e-4)


def test_tiny_loop_terminations():
    """tiny_loop_kernel's tolerance and time-budget stops, through spgm_solve, against the per-iteration path."""
    scn = configs.small_scenario()
    rng = np.random.default_rng(5)
    s_true = np.zeros(scn.n_voxels, complex)
    s_true[rng.choice(scn.n_voxels, 5, replace=False)] = 1.0
    from paper_2509_00774_b200 import forward_apply, lipschitz_estimate

    y = forward_apply(s_true, scn)
    eta = 0.9 / lipschitz_estimate(scn, n_iters=50)
    cfg = SolverConfig(eta=eta, alpha=1e-6, tol=2e-3, max_iters=500, flat_batch=64, rng_seed=1)
    r1 = spgm_solve(y, scn, cfg)
    import os

    os.environ["NFGPU_LOOP"] = "0"
    try:
        r0 = spgm_solve(y, scn, cfg)
    finally:
        os.environ.pop("NFGPU_LOOP")
    assert r1.termination == r0.termination == "tolerance_reached"
    assert abs(r1.iterations - r0.iterations) <= 1
    assert rel_l2(r1.volume.values, r0.volume.values) <= 1e-9
    rep = spgm_solve(y, scn, SolverConfig(eta=eta, alpha=1e-6, tol=1e-300, max_iters=10_000_000, flat_batch=32,
                                          time_budget_s=0.05))
    assert rep.termination == "time_budget" and 1 <= rep.iterations < 10_000_000


@pytest.mark.parametrize("workload,dtype", [("small", "c128"), ("medium", "c64")])
def test_chained_launches_match_one_launch(workload, dtype, monkeypatch):
    """nf_spgm_loop_chained: launches enqueued back to back (odd and even chunk sizes, so the iterate is folded
    back into s_a after odd counts) give the iterate and records of one launch over the same index table; a launch
    whose predecessor stopped early runs no iteration and forwards the reason."""
    w = configs.WORKLOADS[workload]()
    scn = w.scenario
    rng = np.random.default_rng(8)
    y = rc(rng, scn.n_channels)
    s0 = rc(rng, scn.n_voxels) * 0.01
    a, b = _pair(scn, dtype, y, 1e-3, 1e-7, s0, max_batch=w.batch)
    K = 12
    table = np.stack([np.sort(rng.choice(scn.n_channels, w.batch, replace=False)) for _ in range(K)])
    a.run_loop(K, table=table, tol=0.0)
    assert a.loop_result() == (K, 0)
    rec_a = a._loop_rec[:K, :4].clone()
    sizes, at, slot, prev, recs = [3, 4, 5], 0, 0, None, []
    for n in sizes:
        b.run_loop_chained(slot, prev, n, table=table[at:at + n], tol=0.0)
        prev, slot, at = slot, slot ^ 1, at + n
        k_run, reason, rec = b.chained_result(prev)
        assert (k_run, reason) == (n, 0)
        recs.append(rec[:n, :4].copy())
    assert torch.equal(a.s, b.s)
    assert np.array_equal(np.concatenate(recs), rec_a.cpu().numpy())
    # early stop: a tolerance every iteration meets stops the first launch after one iteration; the next runs none
    c, _ = _pair(scn, dtype, y, 1e-3, 1e-7, s0, max_batch=w.batch)
    c.run_loop_chained(0, None, 4, table=table[:4], tol=1e9)
    c.run_loop_chained(1, 0, 4, table=table[4:8], tol=0.0)
    assert c.chained_result(0)[:2] == (1, 1)
    assert c.chained_result(1)[:2] == (0, 1)
    a2, _ = _pair(scn, dtype, y, 1e-3, 1e-7, s0, max_batch=w.batch)
    a2.run_loop(1, table=table[:1], tol=0.0)
    a2.loop_result()
    assert torch.equal(a2.s, c.s)
