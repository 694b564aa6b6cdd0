#!/usr/bin/env python3
"""Record the REFERENCE geometry layer's outputs (pkg/src/nfmimo/geometry.py) for tests/test_geometry.py:

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_geometry_golden.py

Spiral layouts, voxel centres, channel decoding, frequency grids, pulse interpolation and scenario
fingerprints of the paper-v preset and a few seeded scenarios.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("NFMIMO_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
import nfmimo as ref  # noqa: E402

OUT = Path(__file__).resolve().parent / "geometry.npz"
SPIRALS = [(16, 9, 0.25, 7), (3, 2, 0.15, 3), (5, 4, 0.2, 1), (1, 1, 0.1, 0), (48, 48, 0.3, 11)]


def main():
    out = {}
    for i, (nt, nr, rad, seed) in enumerate(SPIRALS):
        arr = ref.make_spiral_array(nt, nr, rad, rng_seed=seed)
        out[f"spiral{i}_tx"] = np.array([[p.x, p.y, p.z] for p in arr.transmitters])
        out[f"spiral{i}_rx"] = np.array([[p.x, p.y, p.z] for p in arr.receivers])
    pv = ref.preset_scenario("paper-v")
    rng = np.random.default_rng(5)
    ns = rng.choice(pv.n_voxels, 64, replace=False)
    out["pv_voxels"] = ns
    out["pv_centers"] = np.array([[c.x, c.y, c.z] for c in (ref.voxel_center(int(n), pv.voxels) for n in ns)])
    ms = rng.choice(pv.n_channels, 64, replace=False)
    out["pv_channels"] = ms
    out["pv_decoded"] = np.array([[c.fi, c.ti, c.ri] for c in (ref.channel_of(int(m), pv) for m in ms)])
    out["pv_freqs"] = pv.frequencies.values()
    out["pv_fingerprint"] = np.frombuffer(ref.scenario_fingerprint(pv), dtype=np.uint8)
    out["pv_dims"] = np.array([pv.n_channels, pv.n_voxels])
    tab = ref.TabulatedPulse((4e9, 6e9, 8e9), (1 + 0j, 0.5 - 0.25j, 0.1 + 0.3j))
    fq = np.linspace(4e9, 8e9, 17)
    out["pulse_f"] = fq
    out["pulse_v"] = tab.evaluate(fq)
    fg = ref.FrequencyGrid(57e9, 64e9, 128)
    out["fg_values"] = fg.values()
    out["fg_spacing"] = np.array([fg.spacing])
    np.savez(OUT, **out)
    print("wrote", OUT, sorted(out))


if __name__ == "__main__":
    main()
