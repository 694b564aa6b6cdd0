"""CPU: the C-ABI library builds, loads and exports every symbol include/nfgpu.h
declares; host-side validation mirrors the reference's exception types; no
compute call is made without a GPU."""

from __future__ import annotations

import ctypes
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2509_00774_b200 import _build, _lib, geometry as G
from paper_2509_00774_b200.forward import ChannelSubset, MeasurementSet, ReflectivityVolume, _subset_indices
from paper_2509_00774_b200.solver import MinibatchComposition, SolverConfig, sample_minibatch


def header_symbols():
    text = (ROOT / "include" / "nfgpu.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(nf_\w+)\s*\(", text, re.M)))


def test_header_symbols_bound():
    syms = header_symbols()
    assert len(syms) == 21
    assert set(syms) == set(_lib.SIGNATURES)


def test_library_loads_and_exports_all_symbols():
    lib = _lib.load()
    assert _build.LIB.exists()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert isinstance(lib.nf_last_error(), bytes)


def test_library_is_sm100a():
    data = _build.LIB.read_bytes()
    assert b"sm_100a" in data or b"sm_100" in data


def test_plan_create_rejects_bad_args_without_gpu():
    lib = _lib.load()
    out = ctypes.c_void_p()
    z = np.zeros(3)
    p = z.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    dims = (ctypes.c_int * 3)(1, 1, 1)
    rc = lib.nf_plan_create(p, 0, p, 1, p, p, 1, 3e8, p, p, dims, 0, 1, 0, 1, ctypes.byref(out))
    assert rc == _lib.NF_ERR_ARG and b"n_tx" in lib.nf_last_error()
    rc = lib.nf_plan_create(p, 1, p, 1, p, p, 1, -1.0, p, p, dims, 0, 1, 0, 1, ctypes.byref(out))
    assert rc == _lib.NF_ERR_ARG
    rc = lib.nf_plan_create(p, 1, p, 1, p, p, 1, 3e8, p, p, dims, 0, 2, 0, 1, ctypes.byref(out))
    assert rc == _lib.NF_ERR_ARG and b"slab" in lib.nf_last_error()
    with pytest.raises(ValueError):
        _lib.check(_lib.NF_ERR_ARG, "x")


def test_channel_subset_validation(small_scenario):
    with pytest.raises(ValueError):
        ChannelSubset(np.array([], dtype=int))
    with pytest.raises(ValueError):
        ChannelSubset(np.array([1, 2, 1]))
    with pytest.raises(ValueError):
        ChannelSubset(np.array([-1, 0]))
    assert ChannelSubset(np.array([5, 1, 3])).indices.tolist() == [5, 1, 3]
    with pytest.raises(IndexError):
        _subset_indices(np.array([small_scenario.n_channels]), small_scenario)


def test_domain_type_validation(tiny_scenario, small_scenario):
    with pytest.raises(ValueError):
        ReflectivityVolume(np.zeros(3, dtype=complex), tiny_scenario.voxels)
    bad = np.zeros(tiny_scenario.n_voxels, dtype=complex)
    bad[0] = np.inf
    with pytest.raises(ValueError):
        ReflectivityVolume(bad, tiny_scenario.voxels)
    with pytest.raises(ValueError, match="fingerprint"):
        MeasurementSet(np.zeros(4, dtype=complex), b"short")
    with pytest.raises(ValueError, match="noise_sigma"):
        MeasurementSet(np.zeros(4, dtype=complex), bytes(32), noise_sigma=-2.0)
    ms = MeasurementSet.for_scenario(np.zeros(tiny_scenario.n_channels, dtype=complex), tiny_scenario)
    assert ms.matches(tiny_scenario) and not ms.matches(small_scenario)


def test_geometry_validation_and_index_maps(small_scenario):
    with pytest.raises(ValueError):
        G.ArrayGeometry(((0, 0, 0.1),), ((0, 0, 0),))
    with pytest.raises(ValueError):
        G.ArrayGeometry(((0, 0, 0), (0, 0, 0)), ((1, 0, 0),))
    with pytest.raises(ValueError):
        G.FrequencyGrid(1e9, 2e9, 1)
    with pytest.raises(ValueError):
        G.VoxelGrid((0, 0, 1), (0.1, 0, 0), (1, 1, 1))
    with pytest.raises(G.SingularityError):
        G.ImagingScenario(
            array=G.ArrayGeometry(((0, 0, 0),), ((0.3, 0, 0),)),
            frequencies=G.FrequencyGrid(1e9, 1e9, 1),
            voxels=G.VoxelGrid((0, 0, 0), (0.2, 0.2, 0), (3, 3, 1)),
        )
    scn = small_scenario
    for m in range(scn.n_channels):
        assert G.flat_channel(G.channel_of(m, scn), scn) == m
    for n in range(scn.n_voxels):
        assert scn.voxels.flat_index(*scn.voxels.indices_of(n)) == n
    assert np.allclose(np.array([G.voxel_center(n, scn.voxels).as_array() for n in range(scn.n_voxels)]),
                       G.voxel_centers(scn.voxels), rtol=0, atol=0)


def test_solver_config_validation():
    for kw in ({"eta": 0.0}, {"eta": -1.0}, {"alpha": -1e-9}, {"max_iters": 0}, {"tol": 0.0},
               {"time_budget_s": 0.0}, {"threads": 0}, {"sampler": "x"}, {"check_every": 0}):
        with pytest.raises(ValueError):
            SolverConfig(**kw)
    with pytest.raises(ValueError):
        SolverConfig(flat_batch=4, composition=MinibatchComposition(1, 1, 1))
    cfg = SolverConfig()
    assert cfg.eta == 1e-3 and cfg.alpha == 4e-5 and cfg.tol == 1e-3


def test_structured_sampler_matches_reference_sequence(small_scenario):
    g = np.load(ROOT / "tests" / "golden" / "unit_scenarios.npz")
    sub = sample_minibatch(MinibatchComposition(2, 2, 1), small_scenario, np.random.default_rng(9))
    assert np.array_equal(sub.indices, g["small_structured_first_batch"])
    full = sample_minibatch(MinibatchComposition(3, 3, 2), small_scenario, np.random.default_rng(0))
    assert np.array_equal(full.indices, np.arange(small_scenario.n_channels))
    with pytest.raises(ValueError, match="exceeds"):
        sample_minibatch(MinibatchComposition(4, 1, 1), small_scenario, np.random.default_rng(0))


def test_workload_shapes():
    from paper_2509_00774_b200 import configs

    s, md, lg = (configs.WORKLOADS[k]() for k in ("small", "medium", "large"))
    assert (s.scenario.n_channels, s.scenario.n_voxels) == (256, 2048)
    assert (md.scenario.n_channels, md.scenario.n_voxels) == (16384, 131072)
    assert (lg.scenario.n_channels, lg.scenario.n_voxels) == (294912, 1048576)
    mu = configs.micro_scenario("64^3")
    assert mu.n_channels == 1048576 and mu.n_voxels == 64**3
