"""Matrix-free observation operator — public API of the reference's
``nfmimo.forward`` (pkg/src/nfmimo/forward.py), executed by the sm_100a kernels.

Same names, argument meaning, validation order and exception types as the
reference. The numbers come from the GPU:

* ``forward_apply(s, scenario, subset=None, threads=1)``  → forward.py:342-350
* ``adjoint_apply(r, scenario, subset=None, threads=1)``  → forward.py:353-359
* ``simulate_measurements``                                → forward.py:362-386
* ``matrix_element`` / ``materialize_dense``               → forward.py:158-177

Inputs and outputs are numpy complex128 arrays, as in the reference. ``threads``
is accepted and ignored (the GPU result does not depend on it, so the reference's
thread-count agreement contract holds trivially). The extra keyword ``dtype``
selects "c128" (default; fp64 end to end, parity ≤1e-10) or "c64" (fp32 entries
with fp64 phase anchors; the performance mode, parity ≤1e-5). The environment
variable NFGPU_DTYPE changes the default.

Restricting to a subset is bit-exact to slicing the full result. Each channel's
value is produced by the same fixed reduction tree whatever else is in the batch.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from .geometry import (
    ImagingScenario,
    VoxelGrid,
    channel_of,
    scenario_fingerprint,
    voxel_center,
)
from .plan import DevicePlan, cached_plan, require_cuda

__all__ = [
    "ReflectivityVolume",
    "MeasurementSet",
    "ChannelSubset",
    "DenseCapError",
    "matrix_element",
    "forward_apply",
    "adjoint_apply",
    "simulate_measurements",
    "materialize_dense",
    "get_plan",
    "default_dtype",
]


def default_dtype() -> str:
    return os.environ.get("NFGPU_DTYPE", "c128")


def get_plan(scenario: ImagingScenario, dtype: str | None = None, device=None) -> DevicePlan:
    dev = require_cuda(device)
    return cached_plan(scenario, dtype or default_dtype(), dev.index)


class DenseCapError(RuntimeError):
    """Dense materialization would exceed the entry cap."""


@dataclass(eq=False)
class ReflectivityVolume:
    """Complex reflectivity per voxel in flat x-fastest order (forward.py:59-80)."""

    values: np.ndarray
    grid: VoxelGrid

    def __post_init__(self):
        v = np.asarray(self.values, dtype=np.complex128)
        if v.ndim != 1:
            raise ValueError(f"volume values must be 1-D, got shape {v.shape}")
        if v.size != self.grid.n_voxels:
            raise ValueError(f"volume has {v.size} values but grid holds {self.grid.n_voxels} voxels")
        if not np.isfinite(v).all():
            raise ValueError("volume values must be finite")
        self.values = v

    @classmethod
    def zeros(cls, grid: VoxelGrid) -> "ReflectivityVolume":
        return cls(np.zeros(grid.n_voxels, dtype=np.complex128), grid)


@dataclass(eq=False)
class MeasurementSet:
    """Measurements plus the fingerprint of the producing scenario (forward.py:83-115)."""

    values: np.ndarray
    fingerprint: bytes
    noise_sigma: float | None = None

    def __post_init__(self):
        v = np.asarray(self.values, dtype=np.complex128)
        if v.ndim != 1:
            raise ValueError(f"measurement values must be 1-D, got shape {v.shape}")
        self.values = v
        if len(self.fingerprint) != 32:
            raise ValueError("fingerprint must be 32 bytes")
        if self.noise_sigma is not None:
            s = float(self.noise_sigma)
            if not (math.isfinite(s) and s >= 0):
                raise ValueError(f"noise_sigma must be >= 0, got {s}")
            self.noise_sigma = s

    def matches(self, scenario: ImagingScenario) -> bool:
        return self.values.size == scenario.n_channels and self.fingerprint == scenario_fingerprint(scenario)

    @classmethod
    def for_scenario(cls, values, scenario: ImagingScenario, noise_sigma=None) -> "MeasurementSet":
        return cls(values, scenario_fingerprint(scenario), noise_sigma)


@dataclass(eq=False)
class ChannelSubset:
    """Ordered, duplicate-free, non-negative flat channel list (forward.py:118-136)."""

    indices: np.ndarray

    def __post_init__(self):
        idx = np.asarray(self.indices, dtype=np.int64).ravel()
        if idx.size == 0:
            raise ValueError("channel subset must be non-empty")
        if (idx < 0).any():
            raise ValueError("channel indices must be non-negative")
        if np.unique(idx).size != idx.size:
            raise ValueError("channel subset contains duplicates")
        idx.setflags(write=False)
        self.indices = idx

    def __len__(self) -> int:
        return int(self.indices.size)


# ------------------------------------------------------------------ validation


def _volume_values(s, scenario: ImagingScenario) -> np.ndarray:
    if isinstance(s, ReflectivityVolume):
        if s.grid != scenario.voxels:
            raise ValueError("volume grid does not match the scenario voxel grid")
        return s.values
    v = np.asarray(s, dtype=np.complex128)
    if v.shape != (scenario.n_voxels,):
        raise ValueError(f"expected {scenario.n_voxels} voxel values, got shape {v.shape}")
    return v


def _subset_indices(subset, scenario: ImagingScenario) -> np.ndarray:
    if subset is None:
        return np.arange(scenario.n_channels, dtype=np.int64)
    if not isinstance(subset, ChannelSubset):
        subset = ChannelSubset(np.asarray(subset))
    idx = subset.indices
    if (idx >= scenario.n_channels).any():
        raise IndexError(f"channel index {int(idx.max())} out of range [0, {scenario.n_channels})")
    return idx


# ------------------------------------------------------------------ device execution


def _upload(plan: DevicePlan, x: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x)).to(plan.device).to(plan.torch_dtype)


def _stage(plan: DevicePlan, idx: np.ndarray) -> None:
    # Always the flat path: the reference guarantees forward_apply(s, subset=sub) == full[sub]
    # bit for bit (pkg/tests/test_forward.py:142-149), which needs one arithmetic for every subset.
    plan.prepare(torch.from_numpy(idx.astype(np.int32)).to(plan.device))


def forward_values(plan: DevicePlan, values: np.ndarray, idx: np.ndarray) -> np.ndarray:
    s = _upload(plan, values)
    _stage(plan, idx)
    y = plan.forward(s)
    return y.to(torch.complex128).cpu().numpy()


def adjoint_values(plan: DevicePlan, rvals: np.ndarray, idx: np.ndarray) -> np.ndarray:
    r = _upload(plan, rvals)
    _stage(plan, idx)
    g = plan.adjoint(r)
    return g.to(torch.complex128).cpu().numpy()


# ------------------------------------------------------------------ public API


def forward_apply(s, scenario: ImagingScenario, subset=None, threads: int = 1, *, dtype: str | None = None):
    """Entry k is Σ_n A[m_k, n] s_n; subset None means all M channels."""
    values = _volume_values(s, scenario)
    idx = _subset_indices(subset, scenario)
    return forward_values(get_plan(scenario, dtype), values, idx)


def adjoint_apply(r, scenario: ImagingScenario, subset=None, threads: int = 1, *, dtype: str | None = None):
    """Entry n is Σ_k conj(A[m_k, n]) r_k."""
    idx = _subset_indices(subset, scenario)
    rvals = np.asarray(r, dtype=np.complex128)
    if rvals.shape != (idx.size,):
        raise ValueError(f"expected {idx.size} residual values, got shape {rvals.shape}")
    return adjoint_values(get_plan(scenario, dtype), rvals, idx)


def simulate_measurements(s, scenario: ImagingScenario, noise_sigma: float = 0.0, rng_seed: int = 0,
                          threads: int = 1, *, dtype: str | None = None) -> MeasurementSet:
    """y = A s + w with w ~ CN(0, σ²) drawn exactly as the reference does
    (default_rng(seed): Re block then Im block, scaled by σ/√2; forward.py:379-383)."""
    sigma = float(noise_sigma)
    if not (math.isfinite(sigma) and sigma >= 0):
        raise ValueError(f"noise_sigma must be >= 0, got {noise_sigma}")
    y = forward_apply(s, scenario, dtype=dtype)
    if sigma > 0:
        rng = np.random.default_rng(rng_seed)
        m = scenario.n_channels
        noise = rng.standard_normal(m) + 1j * rng.standard_normal(m)
        y = y + (sigma / math.sqrt(2.0)) * noise
    return MeasurementSet(values=y, fingerprint=scenario_fingerprint(scenario), noise_sigma=sigma)


def matrix_element(m: int, n: int, scenario: ImagingScenario, *, dtype: str | None = None) -> complex:
    """A[m, n], evaluated by the GPU forward on the unit volume e_n and channel m."""
    if not 0 <= n < scenario.n_voxels:
        raise IndexError(f"voxel index {n} out of range [0, {scenario.n_voxels})")
    channel_of(m, scenario)  # IndexError for a bad channel, as the reference
    voxel_center(n, scenario.voxels)
    e = np.zeros(scenario.n_voxels, dtype=np.complex128)
    e[n] = 1.0
    return complex(forward_apply(e, scenario, subset=np.array([m]), dtype=dtype)[0])


def materialize_dense(scenario: ImagingScenario, cap: int = 10_000_000, *, dtype: str | None = None) -> np.ndarray:
    """Dense M×N matrix (test oracle only), built column by column on the GPU."""
    m_count, n_count = scenario.n_channels, scenario.n_voxels
    if m_count * n_count > cap:
        raise DenseCapError(f"dense operator would hold {m_count * n_count} entries (cap {cap})")
    plan = get_plan(scenario, dtype)
    _stage(plan, np.arange(m_count, dtype=np.int64))
    out = torch.empty((n_count, m_count), dtype=plan.torch_dtype, device=plan.device)
    e = torch.zeros(n_count, dtype=plan.torch_dtype, device=plan.device)
    for n in range(n_count):
        e.zero_()
        e[n] = 1.0
        plan.forward(e, out=out[n])
    return out.T.to(torch.complex128).cpu().numpy().copy()
