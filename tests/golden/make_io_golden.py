#!/usr/bin/env python3
"""Generate tests/golden/io/ with the REFERENCE's own writers (pkg/src/nfmimo/io.py).

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_io_golden.py

It writes NFMV/NFMS files, scenario JSON documents and CSV slices with the unmodified
reference on seeded inputs, plus inputs.npz holding those inputs. tests/test_io.py checks
that our writers produce the same bytes and our readers decode the reference's files.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("NFMIMO_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
import nfmimo as ref  # noqa: E402
from nfmimo import io as rio  # noqa: E402

OUT = Path(__file__).resolve().parent / "io"


def scenarios():
    tab = ref.ImagingScenario(
        array=ref.ArrayGeometry(transmitters=(ref.Vec3(0.05, 0.0, 0.0), ref.Vec3(-0.05, 0.02, 0.0)),
                                receivers=(ref.Vec3(0.0, 0.04, 0.0),)),
        frequencies=ref.FrequencyGrid(5e9, 7e9, 3),
        voxels=ref.VoxelGrid(center=ref.Vec3(0.0, 0.0, 0.35), extent=(0.1, 0.1, 0.0), dims=(2, 2, 1)),
        pulse=ref.TabulatedPulse((4e9, 6e9, 8e9), (1 + 0j, 0.5 - 0.25j, 0.1 + 0.3j)),
    )
    small = ref.ImagingScenario(
        array=ref.make_spiral_array(3, 2, 0.15, rng_seed=3),
        frequencies=ref.FrequencyGrid(4e9, 9e9, 3),
        voxels=ref.VoxelGrid(center=ref.Vec3(0.0, 0.0, 0.3), extent=(0.12, 0.08, 0.06), dims=(3, 2, 2)),
    )
    return {"tabulated": tab, "small": small, "paper_v": ref.preset_scenario("paper-v")}


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    rng = np.random.default_rng(2024)
    grid = ref.VoxelGrid(center=ref.Vec3(0.01, -0.02, 0.4), extent=(0.1, 0.15, 0.05), dims=(3, 4, 2))
    vol_vals = rng.standard_normal(grid.n_voxels) + 1j * rng.standard_normal(grid.n_voxels)
    vol = ref.ReflectivityVolume(vol_vals, grid)
    rio.write_volume(vol, OUT / "volume.nfmv")
    rio.export_slices_csv(vol, OUT / "slices")
    scns = scenarios()
    small = scns["small"]
    meas_vals = rng.standard_normal(small.n_channels) + 1j * rng.standard_normal(small.n_channels)
    rio.write_measurements(ref.MeasurementSet.for_scenario(meas_vals, small), OUT / "small.nfms")
    for name, scn in scns.items():
        rio.write_scenario(scn, OUT / f"{name}.json")
    # a zero volume and a single voxel (normalisation edge cases)
    g1 = ref.VoxelGrid(center=ref.Vec3(0, 0, 0.3), extent=(0, 0, 0), dims=(1, 1, 1))
    rio.write_volume(ref.ReflectivityVolume(np.array([0.3 - 0.4j]), g1), OUT / "single.nfmv")
    np.savez(OUT / "inputs.npz", volume=vol_vals, measurements=meas_vals,
             fingerprints=np.array([list(ref.scenario_fingerprint(s)) for s in scns.values()], dtype=np.uint8),
             names=np.array(list(scns)))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
