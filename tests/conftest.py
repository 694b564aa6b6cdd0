"""Shared fixtures. GPU tests carry @pytest.mark.gpu and call the CUDA path
through the C ABI; everything else runs on the CPU (oracle pins, host logic,
ABI symbol exports, gloo multi-process sharding)."""

from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402
import pytest  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_2509_00774_b200 import geometry as G  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name: str):
    return np.load(GOLDEN / f"{name}.npz")


def rc(rng, n):
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


def rel_l2(a, b) -> float:
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def tiny() -> G.ImagingScenario:
    """2 f × 2 Tx × 2 Rx = 8 channels, 2×2×1 voxels (the reference tests' tiny fixture)."""
    return G.ImagingScenario(
        array=G.ArrayGeometry(
            transmitters=(G.Vec3(0.05, 0.0, 0.0), G.Vec3(-0.05, 0.02, 0.0)),
            receivers=(G.Vec3(0.0, 0.04, 0.0), G.Vec3(0.01, -0.03, 0.0)),
        ),
        frequencies=G.FrequencyGrid(5e9, 7e9, 2),
        voxels=G.VoxelGrid(center=G.Vec3(0.0, 0.0, 0.35), extent=(0.1, 0.1, 0.0), dims=(2, 2, 1)),
    )


def small() -> G.ImagingScenario:
    """3 f × 3 Tx × 2 Rx = 18 channels, 3×2×2 voxels (spiral array, seed 3)."""
    return G.ImagingScenario(
        array=G.make_spiral_array(3, 2, 0.15, rng_seed=3),
        frequencies=G.FrequencyGrid(4e9, 9e9, 3),
        voxels=G.VoxelGrid(center=G.Vec3(0.0, 0.0, 0.3), extent=(0.12, 0.08, 0.06), dims=(3, 2, 2)),
    )


@pytest.fixture(scope="session")
def tiny_scenario():
    return tiny()


@pytest.fixture(scope="session")
def small_scenario():
    return small()


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
