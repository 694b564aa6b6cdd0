"""The BASELINE.json workloads as scenarios, scenes and seeds.

BASELINE.json names five configurations. The reference ships no builders for
them (its presets are geometry.py:442-456). They are defined here once and used
by bench.py and the tests. Seeds that BASELINE.json leaves open are fixed in
``SEEDS``: array 0, scene 0, noise 1, power iteration 0,
minibatch 0. No public dataset is involved. Every input is synthetic and seeded.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .geometry import ArrayGeometry, ConstantPulse, FrequencyGrid, ImagingScenario, Vec3, VoxelGrid

C_BASELINE = 2.998e8  # BASELINE.json uses c = 2.998e8 (the reference default is the SI value)
SEEDS = {"array": 0, "scene": 0, "noise": 1, "power": 0, "minibatch": 0}


@dataclass(frozen=True)
class Workload:
    name: str
    scenario: ImagingScenario
    batch: int            # flat minibatch size |B|
    iters: int            # SPGM iterations
    snr_db: float
    dtype: str
    n_scatterers: int
    l_patch: bool = False


def small_scenario() -> ImagingScenario:
    xs = (-0.06, -0.02, 0.02, 0.06)
    return ImagingScenario(
        array=ArrayGeometry(tuple(Vec3(x, 0.08, 0.0) for x in xs), tuple(Vec3(x, -0.08, 0.0) for x in xs)),
        frequencies=FrequencyGrid(60e9, 64e9, 16),
        voxels=VoxelGrid(center=Vec3(0.0, 0.0, 0.30), extent=(0.2, 0.2, 0.1), dims=(16, 16, 8)),
        pulse=ConstantPulse(1.0),
        c=C_BASELINE,
    )


def medium_scenario(seed: int = SEEDS["array"]) -> ImagingScenario:
    rng = np.random.default_rng(seed)
    tx = rng.uniform(-0.15, 0.15, size=(16, 2))
    rx = rng.uniform(-0.15, 0.15, size=(16, 2))
    return ImagingScenario(
        array=ArrayGeometry(tuple(Vec3(a, b, 0.0) for a, b in tx), tuple(Vec3(a, b, 0.0) for a, b in rx)),
        frequencies=FrequencyGrid(57e9, 64e9, 64),
        voxels=VoxelGrid(center=Vec3(0.0, 0.0, 0.40), extent=(0.3, 0.3, 0.2), dims=(64, 64, 32)),
        pulse=ConstantPulse(1.0),
        c=C_BASELINE,
    )


def _line_array(n_tx: int, n_rx: int, half: float, seed: int) -> ArrayGeometry:
    """Tx on y = ±half with seeded x; Rx on x = ±half with seeded y (BASELINE 'Large')."""
    rng = np.random.default_rng(seed)
    h = n_tx // 2
    tx_x = rng.uniform(-half, half, size=n_tx)
    rx_y = rng.uniform(-half, half, size=n_rx)
    tx = [Vec3(tx_x[i], half if i < h else -half, 0.0) for i in range(n_tx)]
    g = n_rx // 2
    rx = [Vec3(half if i < g else -half, rx_y[i], 0.0) for i in range(n_rx)]
    return ArrayGeometry(tuple(tx), tuple(rx))


def large_scenario(seed: int = SEEDS["array"]) -> ImagingScenario:
    return ImagingScenario(
        array=_line_array(48, 48, 0.2, seed),
        frequencies=FrequencyGrid(57e9, 64e9, 128),
        voxels=VoxelGrid(center=Vec3(0.0, 0.0, 0.45), extent=(0.4, 0.4, 0.3), dims=(128, 128, 64)),
        pulse=ConstantPulse(1.0),
        c=C_BASELINE,
    )


def micro_scenario(grid: str = "128^3", seed: int = SEEDS["array"]) -> ImagingScenario:
    """Operator microbenchmark: the Large layout with 64 Tx / 64 Rx and 256 frequencies
    (M = 1,048,576) over the Large extent, grids 64³, 128³ or 192×192×96."""
    dims = {"64^3": (64, 64, 64), "128^3": (128, 128, 128), "192x192x96": (192, 192, 96)}[grid]
    return ImagingScenario(
        array=_line_array(64, 64, 0.2, seed),
        frequencies=FrequencyGrid(57e9, 64e9, 256),
        voxels=VoxelGrid(center=Vec3(0.0, 0.0, 0.45), extent=(0.4, 0.4, 0.3), dims=dims),
        pulse=ConstantPulse(1.0),
        c=C_BASELINE,
    )


WORKLOADS = {
    "small": lambda: Workload("small", small_scenario(), 32, 200, 30.0, "c128", 20),
    "medium": lambda: Workload("medium", medium_scenario(), 512, 300, 30.0, "c64", 200, l_patch=True),
    "large": lambda: Workload("large", large_scenario(), 4096, 500, 25.0, "c64", 1000),
}


def make_scene(w: Workload, seed: int = SEEDS["scene"]) -> np.ndarray:
    """Seeded sparse scene: k scatterers at distinct random voxels, |s| ~ U[0.5, 1],
    arg s ~ U[0, 2π); Medium adds an L-shaped unit-amplitude random-phase patch in
    the middle z-plane (two orthogonal bars)."""
    scn = w.scenario
    N = scn.n_voxels
    rng = np.random.default_rng(seed)
    s = np.zeros(N, dtype=np.complex128)
    pos = rng.choice(N, w.n_scatterers, replace=False)
    amp = rng.uniform(0.5, 1.0, size=w.n_scatterers)
    ph = rng.uniform(0.0, 2.0 * math.pi, size=w.n_scatterers)
    s[pos] = amp * np.exp(1j * ph)
    if w.l_patch:
        nx, ny, nz = scn.voxels.dims
        iz = nz // 2
        x0, y0, L = nx // 4, ny // 4, nx // 2
        cells = [(x0 + i, y0) for i in range(L)] + [(x0, y0 + j) for j in range(1, L)]
        for ix, iy in cells:
            s[ix + nx * (iy + ny * iz)] = np.exp(1j * rng.uniform(0.0, 2.0 * math.pi))
    return s


def noise_sigma(clean: np.ndarray, snr_db: float) -> float:
    """σ with mean|A s|²/σ² = SNR (the reference's recipe, run_minibatch_study.py:54)."""
    return float(np.sqrt(np.mean(np.abs(clean) ** 2) * 10 ** (-snr_db / 10)))


def add_noise(clean: np.ndarray, sigma: float, seed: int = SEEDS["noise"]) -> np.ndarray:
    """y = clean + σ/√2 (N + jN) with default_rng(seed), as forward.py:379-383."""
    if sigma <= 0:
        return clean.copy()
    rng = np.random.default_rng(seed)
    m = clean.size
    return clean + (sigma / math.sqrt(2.0)) * (rng.standard_normal(m) + 1j * rng.standard_normal(m))
