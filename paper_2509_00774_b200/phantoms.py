"""Synthetic scenes for `simulate` (pkg/src/nfmimo/phantoms.py).

Specs: ``points:k`` (k unit scatterers at distinct random voxels with random phases, drawn
from default_rng(seed) as the reference: the voxel choice first, then the phases),
``bar`` (unit voxels along x through the centre, x in [nx/4, 3nx/4]), ``cross`` (the bar
plus the same along y in the central z plane), and ``file:path`` (a volume file whose dims
must match the grid).
"""

from __future__ import annotations

import numpy as np

from .forward import ReflectivityVolume
from .geometry import VoxelGrid

__all__ = ["make_phantom", "PHANTOM_KINDS"]

PHANTOM_KINDS = ("points", "bar", "cross", "file")


def _line(grid: VoxelGrid, values: np.ndarray, axis: int) -> None:
    nx, ny, nz = grid.dims
    n = (nx, ny)[axis]
    for i in range(n // 4, 3 * n // 4 + 1):
        ix, iy = (i, ny // 2) if axis == 0 else (nx // 2, i)
        values[grid.flat_index(ix, iy, nz // 2)] = 1.0


def make_phantom(spec: str, grid: VoxelGrid, rng_seed: int = 0) -> ReflectivityVolume:
    spec = spec.strip()
    values = np.zeros(grid.n_voxels, dtype=np.complex128)
    if spec.startswith("points:"):
        k = int(spec.split(":", 1)[1])
        if k < 1:
            raise ValueError(f"points phantom needs k >= 1, got {k}")
        if k > grid.n_voxels:
            raise ValueError(f"cannot place {k} scatterers in {grid.n_voxels} voxels")
        rng = np.random.default_rng(rng_seed)
        sites = rng.choice(grid.n_voxels, size=k, replace=False)
        values[sites] = np.exp(1j * rng.uniform(0.0, 2.0 * np.pi, size=k))
        return ReflectivityVolume(values, grid)
    if spec in ("bar", "cross"):
        _line(grid, values, 0)
        if spec == "cross":
            _line(grid, values, 1)
        return ReflectivityVolume(values, grid)
    if spec.startswith("file:"):
        from .io import read_volume

        return read_volume(spec.split(":", 1)[1], grid=grid)
    raise ValueError(f"unknown phantom spec {spec!r}; expected points:k, bar, cross, or file:path")
