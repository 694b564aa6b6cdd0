"""Geometry layer (paper_2509_00774_b200.geometry) on CPU: the domain types' validation, indexing and
layouts, following the reference's geometry test strategy (pkg/tests/test_geometry.py). Values the
reference computes (spiral layouts, voxel centres, channel decoding, frequency grids, pulse
interpolation, fingerprints) are pinned to tests/golden/geometry.npz, written by the reference
itself (tests/golden/make_geometry_golden.py)."""

from __future__ import annotations

import math
from pathlib import Path

import numpy as np
import pytest

from conftest import tiny
from paper_2509_00774_b200 import (
    ArrayGeometry,
    ChannelIndex,
    ConstantPulse,
    FrequencyGrid,
    ImagingScenario,
    SingularityError,
    TabulatedPulse,
    Vec3,
    VoxelGrid,
    channel_of,
    flat_channel,
    make_spiral_array,
    preset_scenario,
    scenario_fingerprint,
    voxel_center,
    voxel_centers,
)

G = np.load(Path(__file__).resolve().parent / "golden" / "geometry.npz")
SPIRALS = [(16, 9, 0.25, 7), (3, 2, 0.15, 3), (5, 4, 0.2, 1), (1, 1, 0.1, 0), (48, 48, 0.3, 11)]
PAPER_GRID = preset_scenario("paper-v").voxels


def xyz(points):
    return np.array([[p.x, p.y, p.z] for p in points])


# ------------------------------------------------------------------ pinned to the reference


@pytest.mark.parametrize("i", range(len(SPIRALS)))
def test_spiral_layouts_match_reference(i):
    nt, nr, rad, seed = SPIRALS[i]
    arr = make_spiral_array(nt, nr, rad, rng_seed=seed)
    assert np.array_equal(xyz(arr.transmitters), G[f"spiral{i}_tx"])
    assert np.array_equal(xyz(arr.receivers), G[f"spiral{i}_rx"])


def test_paper_preset_matches_reference():
    pv = preset_scenario("paper-v")
    assert [pv.n_channels, pv.n_voxels] == G["pv_dims"].tolist() == [1584, 78141]
    assert scenario_fingerprint(pv) == bytes(G["pv_fingerprint"].tolist())
    assert np.array_equal(pv.frequencies.values(), G["pv_freqs"])
    got = np.array([[c.x, c.y, c.z] for c in (voxel_center(int(n), pv.voxels) for n in G["pv_voxels"])])
    assert np.array_equal(got, G["pv_centers"])
    dec = np.array([[c.fi, c.ti, c.ri] for c in (channel_of(int(m), pv) for m in G["pv_channels"])])
    assert np.array_equal(dec, G["pv_decoded"])


def test_pulse_and_frequency_grid_match_reference():
    tab = TabulatedPulse((4e9, 6e9, 8e9), (1 + 0j, 0.5 - 0.25j, 0.1 + 0.3j))
    assert np.array_equal(tab.evaluate(G["pulse_f"]), G["pulse_v"])
    fg = FrequencyGrid(57e9, 64e9, 128)
    assert np.array_equal(fg.values(), G["fg_values"]) and fg.spacing == G["fg_spacing"][0]


# ------------------------------------------------------------------ validation and indexing


def test_vec3_rejects_non_finite():
    for bad in (math.nan, math.inf):
        with pytest.raises(ValueError):
            Vec3(bad, 0.0, 0.0)


def test_array_geometry_validation():
    with pytest.raises(ValueError):
        ArrayGeometry(transmitters=(), receivers=(Vec3(0, 0, 0),))
    with pytest.raises(ValueError, match="z=0"):
        ArrayGeometry(transmitters=(Vec3(0, 0, 0.1),), receivers=(Vec3(0.1, 0, 0),))
    with pytest.raises(ValueError, match="duplicate"):
        ArrayGeometry(transmitters=(Vec3(0, 0, 0), Vec3(0, 0, 0)), receivers=(Vec3(0.1, 0, 0),))


def test_frequency_grid():
    g = FrequencyGrid(4e9, 16e9, 11)
    assert g.spacing == pytest.approx(1.2e9, rel=1e-15)
    v = g.values()
    assert v[0] == 4e9 and v[-1] == 16e9 and v.size == 11
    assert FrequencyGrid(5e9, 5e9, 1).values().tolist() == [5e9]
    for args in [(5e9, 6e9, 1), (0.0, 1e9, 2), (-1e9, 1e9, 2), (2e9, 1e9, 2), (1e9, 2e9, 0)]:
        with pytest.raises(ValueError):
            FrequencyGrid(*args)


def test_voxel_grid_centres_and_indexing():
    assert voxel_center(0, PAPER_GRID) == Vec3(-0.15, -0.15, 0.45)
    assert voxel_center(30 + 61 * (30 + 61 * 10), PAPER_GRID) == Vec3(0.0, 0.0, 0.5)
    v = voxel_center(1, PAPER_GRID)
    assert v.x == pytest.approx(-0.145, abs=1e-15) and (v.y, v.z) == (-0.15, 0.45)
    assert PAPER_GRID.spacing == pytest.approx((0.005, 0.005, 0.005), rel=1e-12)
    for bad in (PAPER_GRID.n_voxels, -1):
        with pytest.raises(IndexError):
            voxel_center(bad, PAPER_GRID)
    for k in (0, 1, 61, 3720, 78140):
        assert PAPER_GRID.flat_index(*PAPER_GRID.indices_of(k)) == k
    with pytest.raises(IndexError):
        PAPER_GRID.flat_index(61, 0, 0)
    centers = voxel_centers(PAPER_GRID)
    assert centers.shape == (78141, 3) and np.unique(centers, axis=0).shape[0] == 78141
    small = VoxelGrid(center=Vec3(0.01, -0.02, 0.3), extent=(0.1, 0.2, 0.0), dims=(3, 4, 1))
    cs = voxel_centers(small)
    for n in range(small.n_voxels):
        assert np.array_equal(cs[n], voxel_center(n, small).as_array())
    for ext, dims in [((0.1, 0.1, 0.1), (2, 2, 1)), ((0.1, 0.0, 0.1), (2, 2, 2))]:
        with pytest.raises(ValueError):
            VoxelGrid(center=Vec3(0, 0, 0), extent=ext, dims=dims)


def test_channel_indexing():
    t = tiny()
    assert channel_of(0, t) == ChannelIndex(0, 0, 0)
    pv = preset_scenario("paper-v")
    assert channel_of(9, pv) == ChannelIndex(fi=0, ti=1, ri=0)
    assert channel_of(144, pv) == ChannelIndex(fi=1, ti=0, ri=0)
    for bad in (t.n_channels, -1):
        with pytest.raises(IndexError):
            channel_of(bad, t)
    with pytest.raises(IndexError):
        flat_channel(ChannelIndex(0, 0, 99), t)
    assert all(flat_channel(channel_of(m, pv), pv) == m for m in range(pv.n_channels))
    rng = np.random.default_rng(1)
    for _ in range(40):
        nf, nt, nr = (int(x) for x in rng.integers(1, 6, size=3))
        scn = ImagingScenario(array=make_spiral_array(nt, nr, 0.2, rng_seed=0),
                              frequencies=FrequencyGrid(1e9, 2e9, nf) if nf > 1 else FrequencyGrid(1e9, 1e9, 1),
                              voxels=VoxelGrid(center=Vec3(0, 0, 0.3), extent=(0, 0, 0), dims=(1, 1, 1)))
        m = int(rng.integers(0, scn.n_channels))
        assert flat_channel(channel_of(m, scn), scn) == m


def test_spiral_array_contract():
    geo = make_spiral_array(16, 9, 0.25, rng_seed=7)
    assert geo.n_tx == 16 and geo.n_rx == 9
    assert all(math.hypot(p.x, p.y) <= 0.25 + 1e-12 and p.z == 0.0 for p in geo.transmitters + geo.receivers)
    g1 = make_spiral_array(1, 1, 0.1, rng_seed=99)
    assert g1.transmitters[0] != g1.receivers[0]
    assert make_spiral_array(5, 4, 0.3, rng_seed=11) == make_spiral_array(5, 4, 0.3, rng_seed=11)
    assert make_spiral_array(5, 4, 0.3, rng_seed=11) != make_spiral_array(5, 4, 0.3, rng_seed=12)
    for radius in (0.0, -0.5, math.nan):
        with pytest.raises(ValueError):
            make_spiral_array(2, 2, radius)


def test_pulse_spectra():
    assert np.all(ConstantPulse(2.0 - 1.0j).evaluate(np.array([1e9, 5e9, 9e9])) == 2.0 - 1.0j)
    p = TabulatedPulse(frequencies_hz=(1e9, 3e9), values=(1 + 0j, 3 + 4j))
    assert p.evaluate(np.array([2e9]))[0] == pytest.approx(2 + 2j, rel=1e-15)
    with pytest.raises(ValueError):
        TabulatedPulse(frequencies_hz=(2e9, 1e9), values=(1 + 0j, 1 + 0j))
    with pytest.raises(ValueError, match="cover"):
        ImagingScenario(array=make_spiral_array(1, 1, 0.1), frequencies=FrequencyGrid(4e9, 8e9, 3),
                        voxels=VoxelGrid(center=Vec3(0, 0, 0.3), extent=(0, 0, 0), dims=(1, 1, 1)),
                        pulse=TabulatedPulse(frequencies_hz=(5e9, 6e9), values=(1 + 0j, 1 + 0j)))


def test_scenario_validation_and_fingerprint():
    with pytest.raises(ValueError):
        preset_scenario("nope")
    with pytest.raises(SingularityError):
        ImagingScenario(array=ArrayGeometry(transmitters=(Vec3(0, 0, 0),), receivers=(Vec3(0.1, 0, 0),)),
                        frequencies=FrequencyGrid(1e9, 1e9, 1),
                        voxels=VoxelGrid(center=Vec3(0, 0, 0), extent=(0, 0, 0), dims=(1, 1, 1)))
    a, b = preset_scenario("paper-v"), preset_scenario("paper-v")
    assert scenario_fingerprint(a) == scenario_fingerprint(b) and len(scenario_fingerprint(a)) == 32
    other = ImagingScenario(array=a.array, frequencies=FrequencyGrid(4e9, 16e9, 12), voxels=a.voxels)
    assert scenario_fingerprint(other) != scenario_fingerprint(a)
