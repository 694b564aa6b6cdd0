"""Metrics (paper_2509_00774_b200.metrics): PSNR over peak-normalised magnitudes, the sweep CSV and
Spearman ranks on CPU, and run_sweep on the GPU solvers, following the reference's metrics test
strategy (pkg/tests/test_metrics.py)."""

from __future__ import annotations

import csv
import math

import numpy as np
import pytest

from conftest import rc, tiny
from paper_2509_00774_b200 import MinibatchComposition, ReflectivityVolume, SolverConfig, Vec3, VoxelGrid
from paper_2509_00774_b200.metrics import (
    SWEEP_CSV_HEADER,
    SweepRecord,
    psnr_vs_reference,
    run_sweep,
    spearman_rank,
    write_sweep_csv,
)

GRID4 = VoxelGrid(center=Vec3(0, 0, 0.3), extent=(0.1, 0, 0), dims=(4, 1, 1))


def vol(values, grid=GRID4):
    return ReflectivityVolume(np.asarray(values, dtype=complex), grid)


def test_psnr_identity_scale_and_hand_value(rng):
    v = vol(rc(rng, 4))
    r = psnr_vs_reference(v, v)
    assert math.isinf(r.psnr_db) and r.rmse == 0.0
    ref = vol(rc(rng, 4))
    r = psnr_vs_reference(vol(ref.values * (3.7 * np.exp(1j * 1.234))), ref)
    assert math.isinf(r.psnr_db) or r.psnr_db > 250.0  # a general complex scale moves magnitudes by ~1 ulp
    mags = np.abs(rc(rng, 4)) + 0.1
    r = psnr_vs_reference(vol(mags), vol(4.0 * mags))  # an exact power of two: exactly infinite
    assert math.isinf(r.psnr_db) and r.rmse == 0.0
    r = psnr_vs_reference(vol([1.0, 0, 0, 0]), vol([1.0, 0.02, 0, 0]))  # rmse = 0.02/2 -> 40 dB
    assert r.rmse == pytest.approx(0.01, rel=1e-12) and r.psnr_db == pytest.approx(40.0, abs=1e-9)


def test_psnr_edge_cases(rng):
    other = VoxelGrid(center=Vec3(0, 0, 0), extent=(0.1, 0, 0), dims=(4, 1, 1))
    with pytest.raises(ValueError, match="grid"):
        psnr_vs_reference(vol(np.ones(4)), vol(np.ones(4), grid=other))
    with pytest.raises(ValueError, match="zero"):
        psnr_vs_reference(vol(np.ones(4)), vol(np.zeros(4)))
    assert psnr_vs_reference(vol(np.zeros(4)), vol([1, 0, 0, 0])).rmse == pytest.approx(0.5)
    a, b = np.abs(rc(rng, 4)), np.abs(rc(rng, 4))
    a, b = a / a.max(), b / b.max()
    assert psnr_vs_reference(vol(a), vol(b)).rmse == pytest.approx(psnr_vs_reference(vol(b), vol(a)).rmse, rel=1e-12)
    mags = np.abs(rc(rng, 4)) + 0.1
    assert psnr_vs_reference(vol(mags), vol(2.0 * mags)).rmse == 0.0
    assert psnr_vs_reference(vol(mags * [1, 1, 1, 1.5]), vol(2.0 * mags)).rmse > 0.0


def test_psnr_scale_invariance_property():
    for seed in range(50):
        rng = np.random.default_rng(seed)
        a, b = vol(rc(rng, 4)), vol(rc(rng, 4))
        base = psnr_vs_reference(a, b)
        c1, c2 = complex(*rng.standard_normal(2)), complex(*rng.standard_normal(2))
        scaled = psnr_vs_reference(vol(a.values * c1), vol(b.values * c2))
        assert scaled.rmse == pytest.approx(base.rmse, rel=1e-9, abs=1e-12)


def test_sweep_csv_header_and_inf_sentinel(tmp_path):
    recs = [SweepRecord(MinibatchComposition(1, 2, 2), seed=7, iterations=12, runtime_s=0.5, psnr_db=math.inf),
            SweepRecord(MinibatchComposition(2, 2, 2), seed=8, iterations=9, runtime_s=1.25, psnr_db=38.75)]
    path = tmp_path / "sweep.csv"
    write_sweep_csv(recs, path)
    rows = list(csv.reader(path.open(newline="")))
    assert rows[0] == SWEEP_CSV_HEADER
    assert rows[1] == ["1", "2", "2", "4", "7", "12", "0.5", "inf"]
    assert rows[2][:6] == ["2", "2", "2", "8", "8", "9"] and float(rows[2][7]) == pytest.approx(38.75)


def test_spearman():
    assert spearman_rank([1, 2, 3, 4], [10, 20, 40, 80]) == pytest.approx(1.0)
    assert spearman_rank([1, 2, 3, 4], [4, 3, 2, 1]) == pytest.approx(-1.0)
    assert spearman_rank([1, 2, 2, 3], [1, 2, 3, 4]) == pytest.approx(0.9486832980505138)
    for bad in (([1], [1]), ([1, 2], [1, 2, 3]), (np.ones((2, 2)), np.ones((2, 2)))):
        with pytest.raises(ValueError):
            spearman_rank(*bad)


# ------------------------------------------------------------------ run_sweep on the GPU solvers


@pytest.mark.gpu
def test_run_sweep_records_and_determinism(rng):
    from paper_2509_00774_b200 import forward_apply

    scn = tiny()
    s = np.zeros(scn.n_voxels, dtype=complex)
    s[1] = 1.0
    y = forward_apply(s, scn)
    assert run_sweep(y, scn, SolverConfig(max_iters=3), [MinibatchComposition(1, 1, 1)], []) == []
    full = run_sweep(y, scn, SolverConfig(max_iters=40, tol=1e-8), [MinibatchComposition(2, 2, 2)], [0])
    assert len(full) == 1 and (math.isinf(full[0].psnr_db) or full[0].psnr_db >= 120.0)
    y = forward_apply(rc(rng, scn.n_voxels), scn)
    comps = [MinibatchComposition(1, 1, 1), MinibatchComposition(2, 2, 2)]
    recs = run_sweep(y, scn, SolverConfig(max_iters=5, tol=1e-30), comps, [3, 4])
    assert [r.seed for r in recs] == [3, 4, 3, 4] and [r.batch_size for r in recs] == [1, 1, 8, 8]
    assert all(r.runtime_s >= 0 and r.iterations == 5 for r in recs)
    comps = [MinibatchComposition(1, 2, 1)]
    a = run_sweep(y, scn, SolverConfig(max_iters=10, tol=1e-30), comps, [5])
    b = run_sweep(y, scn, SolverConfig(max_iters=10, tol=1e-30), comps, [5])
    assert a[0].psnr_db == b[0].psnr_db
