"""Hypothesis property tests mirroring the reference's own: forward subset
consistency (test_forward.py:312-328), prox nonexpansiveness (test_solver.py:220-227), channel
index round trips (test_geometry.py:148-166) and the sampler's composition contract. The
CPU ones run the host logic; the GPU ones run the CUDA path through the C ABI."""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2509_00774_b200 import (
    ArrayGeometry,
    FrequencyGrid,
    ImagingScenario,
    Vec3,
    VoxelGrid,
    channel_of,
    flat_channel,
    make_spiral_array,
)
from paper_2509_00774_b200.solver import MinibatchComposition, sample_minibatch


def _rc(rng, n):
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


@given(nf=st.integers(1, 5), nt=st.integers(1, 5), nr=st.integers(1, 5), data=st.data())
@settings(max_examples=40, deadline=None)
def test_channel_round_trip_property(nf, nt, nr, data):
    scn = ImagingScenario(
        array=make_spiral_array(nt, nr, 0.2, rng_seed=0),
        frequencies=FrequencyGrid(1e9, 2e9, nf) if nf > 1 else FrequencyGrid(1e9, 1e9, 1),
        voxels=VoxelGrid(center=Vec3(0, 0, 0.3), extent=(0, 0, 0), dims=(1, 1, 1)),
    )
    m = data.draw(st.integers(0, scn.n_channels - 1))
    ci = channel_of(m, scn)
    assert flat_channel(ci, scn) == m
    assert m == ci.ri + nr * (ci.ti + nt * ci.fi)  # geometry.py:316-333


@given(nf=st.integers(1, 4), nt=st.integers(1, 5), nr=st.integers(1, 5), seed=st.integers(0, 2**32 - 1))
@settings(max_examples=40, deadline=None)
def test_sample_minibatch_composition_property(nf, nt, nr, seed):
    """solver.py:206-225: a sorted Cartesian product of distinct (f, t, r), B = n_f·n_tx·n_rx."""
    scn = ImagingScenario(
        array=make_spiral_array(5, 5, 0.2, rng_seed=0),
        frequencies=FrequencyGrid(1e9, 2e9, 4),
        voxels=VoxelGrid(center=Vec3(0, 0, 0.3), extent=(0, 0, 0), dims=(1, 1, 1)),
    )
    comp = MinibatchComposition(nf, nt, nr)
    idx = sample_minibatch(comp, scn, np.random.default_rng(seed)).indices
    assert idx.size == comp.batch_size == nf * nt * nr
    assert np.all(np.diff(idx) > 0)
    f, t, r = idx // 25, (idx // 5) % 5, idx % 5
    assert len(set(f)) == nf and len(set(t)) == nt and len(set(r)) == nr


@pytest.mark.gpu
@given(st.integers(0, 2**32 - 1))
@settings(max_examples=15, deadline=None)
def test_forward_subset_consistency_property(seed):
    """The reference's test_forward.py:312-328 scenario: the forward over any subset is bit-exact
    to the same rows of the full forward, on the CUDA path (both precisions)."""
    from paper_2509_00774_b200 import forward_apply

    rng = np.random.default_rng(seed)
    scn = ImagingScenario(
        array=ArrayGeometry(transmitters=(Vec3(0.05, 0, 0), Vec3(-0.04, 0.01, 0)), receivers=(Vec3(0, 0.03, 0),)),
        frequencies=FrequencyGrid(3e9, 5e9, 3),
        voxels=VoxelGrid(center=Vec3(0, 0, 0.25), extent=(0.08, 0, 0.04), dims=(3, 1, 2)),
    )
    s = _rc(rng, scn.n_voxels)
    k = int(rng.integers(1, scn.n_channels + 1))
    sub = np.sort(rng.choice(scn.n_channels, k, replace=False))
    if rng.integers(0, 2):
        sub = sub[::-1].copy()
    for dtype in ("c128", "c64"):
        full = forward_apply(s, scn, dtype=dtype)
        part = forward_apply(s, scn, subset=sub, dtype=dtype)
        assert np.array_equal(part, full[sub])


@pytest.mark.gpu
@given(st.integers(0, 2**32 - 1), st.floats(0, 10))
@settings(max_examples=100, deadline=None)
def test_soft_threshold_nonexpansive_property(seed, alpha):
    """test_solver.py:220-227 on the device prox (nf_soft_threshold)."""
    from paper_2509_00774_b200 import soft_threshold

    rng = np.random.default_rng(seed)
    a, b = _rc(rng, 32), _rc(rng, 32)
    lhs = np.linalg.norm(soft_threshold(a, alpha) - soft_threshold(b, alpha))
    assert lhs <= np.linalg.norm(a - b) * (1 + 1e-12)
