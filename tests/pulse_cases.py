"""Scenarios with a frequency-dependent complex pulse p(f) (TabulatedPulse, reference
geometry.py:239-269), shared by the GPU pulse tests and tests/golden/make_golden.py.

p(f) enters the forward as p_f·Σ (forward.py:150-155, 283-284) and the adjoint as
conj(p_f)·r (forward.py:315-325). Every BASELINE config uses ConstantPulse(1), so these
cases are what exercises the pulse handling of every kernel. Plain parameters only: the
generator rebuilds them with the reference's own types.
"""

from __future__ import annotations

import numpy as np

from paper_2509_00774_b200 import configs
from paper_2509_00774_b200.geometry import (
    ArrayGeometry,
    FrequencyGrid,
    ImagingScenario,
    TabulatedPulse,
    Vec3,
    VoxelGrid,
)


def tabulated_pulse(f_lo: float, f_hi: float, knots: int = 5, seed: int = 0) -> TabulatedPulse:
    """Complex knots (magnitude 0.4-1.6, any phase) spanning slightly more than [f_lo, f_hi]."""
    rng = np.random.default_rng(seed)
    span = f_hi - f_lo if f_hi > f_lo else max(abs(f_lo), 1.0) * 1e-3
    fr = np.linspace(f_lo - 0.05 * span, f_hi + 0.05 * span, knots)
    vals = rng.uniform(0.4, 1.6, knots) * np.exp(1j * rng.uniform(0, 2 * np.pi, knots))
    return TabulatedPulse(tuple(float(f) for f in fr), tuple(complex(v) for v in vals))


def tiny_pulse() -> ImagingScenario:
    return ImagingScenario(
        array=ArrayGeometry((Vec3(0.05, 0.0, 0.0), Vec3(-0.05, 0.02, 0.0)),
                            (Vec3(0.0, 0.04, 0.0), Vec3(0.01, -0.03, 0.0))),
        frequencies=FrequencyGrid(5e9, 7e9, 3),
        voxels=VoxelGrid(center=Vec3(0.0, 0.0, 0.35), extent=(0.1, 0.1, 0.04), dims=(3, 2, 2)),
        pulse=tabulated_pulse(5e9, 7e9, seed=1),
    )


def ragged_pulse() -> ImagingScenario:
    """Odd antenna counts, voxel dims not multiples of the 8x8x4 warp tile."""
    rng = np.random.default_rng(77)
    n_tx, n_rx = 5, 11
    tx = tuple(Vec3(*p) for p in np.c_[rng.uniform(-0.1, 0.1, (n_tx, 2)), np.zeros(n_tx)])
    rx = tuple(Vec3(*p) for p in np.c_[rng.uniform(-0.1, 0.1, (n_rx, 2)), np.zeros(n_rx)])
    return ImagingScenario(array=ArrayGeometry(tx, rx), frequencies=FrequencyGrid(57e9, 64e9, 6),
                           voxels=VoxelGrid(center=Vec3(0, 0, 0.35), extent=(0.1, 0.06, 0.05), dims=(13, 6, 5)),
                           pulse=tabulated_pulse(57e9, 64e9, knots=4, seed=2))


def medium_pulse() -> ImagingScenario:
    """BASELINE Medium geometry (16 + 16 antennas, 64 f, 64x64x32 voxels) with a tabulated pulse."""
    base = configs.medium_scenario()
    return ImagingScenario(array=base.array, frequencies=base.frequencies, voxels=base.voxels,
                           pulse=tabulated_pulse(57e9, 64e9, knots=9, seed=3), c=base.c)


CASES = {"tiny": tiny_pulse, "ragged": ragged_pulse, "medium": medium_pulse}
