"""GPU parity of the operator (forward / adjoint) against the reference's outputs
(tests/golden) and the oracle, through the C ABI. Tolerances are the north star's:
relative L2 ≤ 1e-10 in complex128 and ≤ 1e-5 in complex64. Subset restriction
must be bit-exact."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden, rc, rel_l2, small, tiny
from oracle import nfmimo_oracle as O
from paper_2509_00774_b200 import (
    ArrayGeometry,
    ChannelSubset,
    FrequencyGrid,
    ImagingScenario,
    ReflectivityVolume,
    Vec3,
    VoxelGrid,
    adjoint_apply,
    configs,
    forward_apply,
    materialize_dense,
    matrix_element,
    simulate_measurements,
)
from paper_2509_00774_b200.plan import DevicePlan

pytestmark = pytest.mark.gpu
TOL = {"c128": 1e-10, "c64": 1e-5}
DTYPES = ("c128", "c64")


def one_voxel(tx, rx, vox, f):
    return ImagingScenario(
        array=ArrayGeometry((Vec3(*tx),), (Vec3(*rx),)),
        frequencies=FrequencyGrid(f, f, 1),
        voxels=VoxelGrid(center=Vec3(*vox), extent=(0, 0, 0), dims=(1, 1, 1)),
    )


@pytest.mark.parametrize("dtype", DTYPES)
def test_known_answers(dtype):
    ka = golden("known_answers")
    c = 299_792_458.0
    rel = 1e-12 if dtype == "c128" else 1e-6
    val = matrix_element(0, 0, one_voxel((0.1, 0, 0), (-0.1, 0, 0), (0, 0, 0.4), 10e9), dtype=dtype)
    assert val == pytest.approx(complex(ka["golden_element"]), rel=rel)
    assert val == pytest.approx(-0.4677243613935091 + 0.018818304865202827j, rel=rel)
    assert matrix_element(0, 0, one_voxel((0, 0, 0), (0, 0, 0), (0, 0, 0.5), c), dtype=dtype) == pytest.approx(
        1 / np.pi, rel=rel)
    assert matrix_element(0, 0, one_voxel((0, 0, 0), (0, 0, 0), (0, 0, 0.5), c / 4), dtype=dtype) == pytest.approx(
        -1j / np.pi, rel=rel)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("name,builder", [("tiny", tiny), ("small", small)])
def test_reference_fixture_scenarios(name, builder, dtype):
    g = golden("unit_scenarios")
    scn = builder()
    tol = TOL[dtype]
    assert rel_l2(materialize_dense(scn, dtype=dtype), g[f"{name}_dense"]) <= tol
    s, r, sub = g[f"{name}_s"], g[f"{name}_r"], g[f"{name}_sub"]
    assert rel_l2(forward_apply(s, scn, dtype=dtype), g[f"{name}_fwd"]) <= tol
    assert rel_l2(forward_apply(s, scn, subset=sub, dtype=dtype), g[f"{name}_fwd_sub"]) <= tol
    assert rel_l2(adjoint_apply(r, scn, dtype=dtype), g[f"{name}_adj"]) <= tol
    assert rel_l2(adjoint_apply(r[: sub.size], scn, subset=sub, dtype=dtype), g[f"{name}_adj_sub"]) <= tol


@pytest.mark.parametrize("dtype", DTYPES)
def test_subset_restriction_bit_exact(dtype, rng):
    scn = configs.small_scenario()
    s = rc(rng, scn.n_voxels)
    full = forward_apply(s, scn, dtype=dtype)
    for _ in range(6):
        size = int(rng.integers(1, scn.n_channels + 1))
        sub = rng.choice(scn.n_channels, size=size, replace=False)
        assert np.array_equal(forward_apply(s, scn, subset=sub, dtype=dtype), full[sub])
    # order of the subset is the order of the output
    sub = ChannelSubset(np.array([5, 1, 3]))
    assert np.array_equal(forward_apply(s, scn, subset=sub, dtype=dtype), full[[5, 1, 3]])


@pytest.mark.parametrize("dtype", DTYPES)
def test_subset_restriction_bit_exact_medium(dtype):
    """The reference contract forward_apply(s, subset=sub) == forward_apply(s)[sub] bit for bit
    (forward.py:17-18, test_forward.py:142-149) on Medium (512 tiles): the forward's
    two-level reduce uses a segment count fixed by the plan, so the summation tree of a channel
    does not depend on the batch size. Sizes straddle the old span-dependent segment count."""
    scn = configs.medium_scenario()
    rng = np.random.default_rng(21)
    s = rc(rng, scn.n_voxels)
    full = forward_apply(s, scn, dtype=dtype)
    M = scn.n_channels
    for size in (1, 4096, 13044, M):
        sub = rng.choice(M, size=size, replace=False)
        assert np.array_equal(forward_apply(s, scn, subset=sub, dtype=dtype), full[sub]), size
    # the Cartesian full set staged structured is a different arithmetic; forward_apply stays flat
    assert np.array_equal(forward_apply(s, scn, subset=np.arange(M), dtype=dtype), full)


@pytest.mark.parametrize("dtype", DTYPES)
def test_subset_restriction_bit_exact_multi_window(dtype):
    """A Large 1/8 slab whose full channel set spans several forward windows (fwd_chunk < M):
    every subset, in any order and across window boundaries, reproduces the full result's bits."""
    scn = configs.large_scenario()
    rng = np.random.default_rng(22)
    plan = DevicePlan(scn, dtype=dtype, z_range=(0, 8))
    s = plan._as_dev(rc(rng, plan.n_local), plan.n_local, "s")
    M = scn.n_channels
    plan.prepare(torch.arange(M, dtype=torch.int32, device=plan.device))
    full = plan.forward(s).cpu().numpy()
    for size in (1, 3000, 70000, 200000):
        sub = rng.choice(M, size=size, replace=False)
        plan.prepare(torch.from_numpy(sub.astype(np.int32)).to(plan.device))
        assert np.array_equal(plan.forward(s).cpu().numpy(), full[sub]), size


@pytest.mark.parametrize("dtype", DTYPES)
def test_adjoint_identity_over_random_subsets(dtype, rng):
    scn = small()
    m_count = scn.n_channels
    for _ in range(50):
        size = int(rng.integers(1, m_count + 1))
        sub = rng.choice(m_count, size=size, replace=False)
        s = rc(rng, scn.n_voxels)
        r = rc(rng, size)
        as_ = forward_apply(s, scn, subset=sub, dtype=dtype)
        ahr = adjoint_apply(r, scn, subset=sub, dtype=dtype)
        bound = (1e-10 if dtype == "c128" else 1e-5) * (
            np.linalg.norm(as_) * np.linalg.norm(r) + np.linalg.norm(s) * np.linalg.norm(ahr))
        assert abs(np.vdot(r, as_) - np.vdot(ahr, s)) <= bound


@pytest.mark.parametrize("dtype", DTYPES)
def test_linearity_zero_and_unit_vectors(dtype, small_scenario, rng):
    scn = small_scenario
    assert np.array_equal(forward_apply(np.zeros(scn.n_voxels), scn, dtype=dtype), np.zeros(scn.n_channels))
    assert np.array_equal(adjoint_apply(np.zeros(scn.n_channels), scn, dtype=dtype), np.zeros(scn.n_voxels))
    s1, s2 = rc(rng, scn.n_voxels), rc(rng, scn.n_voxels)
    a, b = 0.7 - 0.2j, -1.3 + 0.4j
    lhs = forward_apply(a * s1 + b * s2, scn, dtype=dtype)
    rhs = a * forward_apply(s1, scn, dtype=dtype) + b * forward_apply(s2, scn, dtype=dtype)
    assert rel_l2(lhs, rhs) <= (1e-12 if dtype == "c128" else 1e-5)
    dense = golden("unit_scenarios")["small_dense"]
    e = np.zeros(scn.n_voxels, complex)
    e[5] = 1.0
    assert rel_l2(forward_apply(e, scn, dtype=dtype), dense[:, 5]) <= TOL[dtype]
    r = np.zeros(scn.n_channels, complex)
    r[7] = 1.0
    assert rel_l2(adjoint_apply(r, scn, dtype=dtype), np.conj(dense[7])) <= TOL[dtype]


def test_validation_errors(small_scenario, tiny_scenario):
    scn = small_scenario
    with pytest.raises(ValueError, match="grid"):
        forward_apply(ReflectivityVolume.zeros(tiny_scenario.voxels), scn)
    with pytest.raises(ValueError, match="voxel values"):
        forward_apply(np.zeros(3), scn)
    with pytest.raises(ValueError, match="residual"):
        adjoint_apply(np.zeros(3), scn, subset=np.array([0, 1]))
    with pytest.raises(IndexError):
        forward_apply(np.zeros(scn.n_voxels), scn, subset=np.array([scn.n_channels]))
    with pytest.raises(ValueError):
        forward_apply(np.zeros(scn.n_voxels), scn, subset=np.array([], dtype=int))
    with pytest.raises(IndexError):
        matrix_element(0, scn.n_voxels, scn)
    with pytest.raises(IndexError):
        matrix_element(scn.n_channels, 0, scn)


@pytest.mark.parametrize("dtype", DTYPES)
def test_baseline_small_probe(dtype):
    b = golden("baseline_small")
    scn = configs.small_scenario()
    assert rel_l2(forward_apply(b["probe_s"], scn, subset=b["probe_idx"], dtype=dtype), b["probe_fwd"]) <= TOL[dtype]
    assert rel_l2(adjoint_apply(b["probe_r"], scn, subset=b["probe_idx"], dtype=dtype), b["probe_adj"]) <= TOL[dtype]
    assert rel_l2(forward_apply(b["s_true"], scn, dtype=dtype), b["clean"]) <= TOL[dtype]


@pytest.mark.parametrize("dtype", DTYPES)
def test_medium_against_reference_outputs(dtype):
    """BASELINE config 1 geometry: the reference's cached-table results (tests/golden/medium_ops.npz)."""
    m = golden("medium_ops")
    scn = configs.medium_scenario()
    s = rc(np.random.default_rng(int(m["s_seed"])), scn.n_voxels)
    r = rc(np.random.default_rng(int(m["r_seed"])), m["idx"].size)
    assert rel_l2(forward_apply(s, scn, subset=m["idx"], dtype=dtype), m["fwd"]) <= TOL[dtype]
    adj = adjoint_apply(r, scn, subset=m["idx"], dtype=dtype)
    assert rel_l2(adj[m["adj_probe_voxels"]], m["adj_probe"]) <= TOL[dtype]
    assert np.linalg.norm(adj) == pytest.approx(float(m["adj_norm"]), rel=TOL[dtype])


def test_large_spot_check_against_direct_formula():
    """BASELINE config 2 (Large, c64): the reference's tables (206 GB) cannot be built, so sampled
    output rows (forward) and sampled voxels (adjoint) are checked against the table-free oracle."""
    scn = configs.large_scenario()
    geo = O.geom_from_scenario(scn)
    rng = np.random.default_rng(5)
    s = rc(rng, scn.n_voxels).astype(np.complex64).astype(np.complex128)
    idx = np.sort(rng.choice(scn.n_channels, 4096, replace=False))
    y = forward_apply(s, scn, subset=idx, dtype="c64")
    rows = rng.choice(idx.size, 24, replace=False)
    assert rel_l2(y[rows], O.direct_forward(geo, s, idx[rows], chunk=65536)) <= 1e-5
    r = rc(rng, idx.size).astype(np.complex64).astype(np.complex128)
    g = adjoint_apply(r, scn, subset=idx, dtype="c64")
    vox = rng.choice(scn.n_voxels, 2048, replace=False)
    assert rel_l2(g[vox], O.direct_adjoint(geo, r, idx, voxels=vox)) <= 1e-5


@pytest.mark.parametrize("dims", [(5, 3, 2), (1, 1, 7), (9, 1, 1), (17, 6, 5), (10, 3, 2), (24, 9, 5)])
def test_ragged_grids_match_oracle(dims, rng):
    """Grids that do not fill the 8×8×4 warp tiles (masked lanes); even nx that is not a multiple of 8 mixes
    lanes on the 16-byte vector path with lanes on the per-voxel path."""
    ext = tuple(0.0 if d == 1 else 0.05 * d / 4 for d in dims)
    scn = ImagingScenario(
        array=ArrayGeometry(((0.03, 0.01, 0.0), (-0.02, 0.04, 0.0), (0.0, -0.05, 0.0)),
                            ((0.01, 0.0, 0.0), (-0.04, -0.01, 0.0))),
        frequencies=FrequencyGrid(20e9, 30e9, 5),
        voxels=VoxelGrid(center=Vec3(0.0, 0.0, 0.3), extent=ext, dims=dims),
    )
    geo = O.geom_from_scenario(scn)
    s, r = rc(rng, scn.n_voxels), rc(rng, scn.n_channels)
    for dtype in DTYPES:
        assert rel_l2(forward_apply(s, scn, dtype=dtype), O.direct_forward(geo, s, np.arange(geo.M))) <= TOL[dtype]
        assert rel_l2(adjoint_apply(r, scn, dtype=dtype), O.direct_adjoint(geo, r, np.arange(geo.M))) <= TOL[dtype]


def test_many_transmitters_several_tx_groups(rng):
    """T=30 (3 shared-memory tx groups in c64, 5 in c128), single-channel and full batches."""
    tx = tuple((0.01 * i - 0.15, 0.07 * ((i % 3) - 1), 0.0) for i in range(30))
    rx = tuple((0.05 * ((i % 2) * 2 - 1), 0.013 * i - 0.05, 0.0) for i in range(9))
    scn = ImagingScenario(array=ArrayGeometry(tx, rx), frequencies=FrequencyGrid(30e9, 32e9, 3),
                          voxels=VoxelGrid(center=Vec3(0, 0, 0.25), extent=(0.05, 0.04, 0.03), dims=(12, 9, 6)))
    geo = O.geom_from_scenario(scn)
    s = rc(rng, scn.n_voxels)
    full = np.arange(geo.M)
    ref_f = O.direct_forward(geo, s, full)
    for dtype in DTYPES:
        assert rel_l2(forward_apply(s, scn, dtype=dtype), ref_f) <= TOL[dtype]
        one = forward_apply(s, scn, subset=[437], dtype=dtype)
        assert abs(one[0] - ref_f[437]) <= TOL[dtype] * 10 * abs(ref_f[437])
        r = rc(rng, 7)
        sub = rng.choice(geo.M, 7, replace=False)
        assert rel_l2(adjoint_apply(r, scn, subset=sub, dtype=dtype), O.direct_adjoint(geo, r, sub)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", DTYPES)
def test_slab_plans_sum_to_full(dtype, rng):
    """Voxel-slab sharding: per-slab forward partials sum to the full forward;
    per-slab adjoints are the slices of the full adjoint."""
    scn = configs.small_scenario()
    s = rc(rng, scn.n_voxels)
    idx = torch.from_numpy(np.sort(rng.choice(scn.n_channels, 40, replace=False)).astype(np.int32)).cuda()
    full = DevicePlan(scn, dtype=dtype)
    full.prepare(idx)
    st = full._as_dev(s, scn.n_voxels, "s")
    y_full = full.forward(st).cpu().numpy()
    r = full._as_dev(rc(rng, 40), 40, "r")
    g_full = full.adjoint(r).cpu().numpy()
    nxy = 16 * 16
    acc = np.zeros_like(y_full)
    for z0, z1 in ((0, 3), (3, 8)):
        p = DevicePlan(scn, dtype=dtype, z_range=(z0, z1))
        p.prepare(idx)
        acc += p.forward(st[z0 * nxy:z1 * nxy].contiguous()).cpu().numpy()
        assert rel_l2(p.adjoint(r).cpu().numpy(), g_full[z0 * nxy:z1 * nxy]) <= TOL[dtype]
    assert rel_l2(acc, y_full) <= TOL[dtype]


def test_simulate_measurements_noise_convention(small_scenario, rng):
    s = rc(rng, small_scenario.n_voxels)
    a = simulate_measurements(s, small_scenario, noise_sigma=0.0)
    assert np.array_equal(a.values, forward_apply(s, small_scenario)) and a.matches(small_scenario)
    b = simulate_measurements(s, small_scenario, noise_sigma=0.5, rng_seed=9)
    c = simulate_measurements(s, small_scenario, noise_sigma=0.5, rng_seed=9)
    assert np.array_equal(b.values, c.values)


@pytest.mark.parametrize("dtype", DTYPES)
def test_microbenchmark_full_M_spot_check(dtype, structured=False):
    """BASELINE config 4 (operator microbenchmark): one forward and one adjoint at full
    M = 64 Tx x 64 Rx x 256 f = 1,048,576 on the 64^3 grid, N(0,1) complex inputs; sampled
    output rows / voxels against the table-free oracle (precision study: c64 and c128)."""
    scn = configs.micro_scenario("64^3")
    geo = O.geom_from_scenario(scn)
    rng = np.random.default_rng(11)
    dt = np.complex64 if dtype == "c64" else np.complex128
    s = rc(rng, scn.n_voxels).astype(dt).astype(np.complex128)
    r = rc(rng, scn.n_channels).astype(dt).astype(np.complex128)
    plan = DevicePlan(scn, dtype=dtype)
    if structured:
        plan.prepare_full()
        assert plan.staged_structured
    else:
        plan.prepare(torch.arange(scn.n_channels, dtype=torch.int32, device=plan.device))
    y = plan.forward(plan._as_dev(s, scn.n_voxels, "s")).to(torch.complex128).cpu().numpy()
    rows = np.sort(rng.choice(scn.n_channels, 16, replace=False))
    assert rel_l2(y[rows], O.direct_forward(geo, s, rows, chunk=32768)) <= TOL[dtype]
    g = plan.adjoint(plan._as_dev(r, scn.n_channels, "r")).to(torch.complex128).cpu().numpy()
    vox = np.sort(rng.choice(scn.n_voxels, 8, replace=False))
    ref = np.concatenate([O.direct_adjoint(geo, r[a:a + 131072], np.arange(a, min(a + 131072, scn.n_channels)),
                                           voxels=vox) for a in range(0, scn.n_channels, 131072)])
    ref = ref.reshape(-1, vox.size).sum(axis=0)
    assert rel_l2(g[vox], ref) <= TOL[dtype]


@pytest.mark.parametrize("dtype", DTYPES)
def test_microbenchmark_full_M_structured_spot_check(dtype):
    """The same full-M microbenchmark through the separable kernels (the full set is Cartesian)."""
    test_microbenchmark_full_M_spot_check(dtype, structured=True)


def test_large_batch_paths_agree():
    """|B| = M (ISTA) on Medium goes through the chunked forward window and the chunked adjoint;
    its result equals the concatenation of smaller batches (forward) and their sum (adjoint)."""
    scn = configs.medium_scenario()
    rng = np.random.default_rng(12)
    s = rc(rng, scn.n_voxels)
    M = scn.n_channels
    y_full = forward_apply(s, scn, dtype="c64")
    parts = [forward_apply(s, scn, subset=np.arange(a, min(a + 4096, M)), dtype="c64") for a in range(0, M, 4096)]
    assert np.array_equal(np.concatenate(parts), y_full)  # subset restriction is bit-exact
    r = rc(rng, M)
    g_full = adjoint_apply(r, scn, dtype="c64")
    g_sum = sum(adjoint_apply(r[a:a + 4096], scn, subset=np.arange(a, min(a + 4096, M)), dtype="c64")
                for a in range(0, M, 4096))
    assert rel_l2(g_full, g_sum) <= 1e-5


@pytest.mark.parametrize("dims", [(10, 3, 2), (24, 9, 5), (17, 6, 5)])
@pytest.mark.parametrize("dtype", DTYPES)
def test_ragged_grid_spgm_step_matches_oracle(dims, dtype, rng):
    """One fused SPGM step (forward, adjoint + prox, statistics) on ragged grids: the prox epilogue's
    vector and per-voxel paths against the oracle's soft_threshold(s - eta * grad)."""
    from paper_2509_00774_b200.solver import SPGMEngine

    ext = tuple(0.05 * d / 4 for d in dims)
    scn = ImagingScenario(
        array=ArrayGeometry(((0.03, 0.01, 0.0), (-0.02, 0.04, 0.0), (0.0, -0.05, 0.0)),
                            ((0.01, 0.0, 0.0), (-0.04, -0.01, 0.0))),
        frequencies=FrequencyGrid(20e9, 30e9, 5),
        voxels=VoxelGrid(center=Vec3(0.0, 0.0, 0.3), extent=ext, dims=dims),
    )
    geo = O.geom_from_scenario(scn)
    s, y = rc(rng, scn.n_voxels), rc(rng, scn.n_channels)
    idx = np.sort(rng.choice(scn.n_channels, 20, replace=False))
    eta, alpha = 2e-3, 0.4
    plan = DevicePlan(scn, dtype=dtype, device="cuda:0")
    eng = SPGMEngine(plan, y, eta=eta, alpha=alpha, initial=s)
    eng.stage(idx)
    eng.step_staged()
    grad = O.direct_adjoint(geo, O.direct_forward(geo, s, idx) - y[idx], idx) / idx.size
    ref = O.soft_threshold(s - eta * grad, alpha)
    assert np.count_nonzero(ref) not in (0, ref.size)  # the threshold is active on some voxels, not all
    assert rel_l2(eng.volume(), ref) <= TOL[dtype]
    assert eng.magnitude_change() == pytest.approx(O.relative_magnitude_change(s, ref), rel=1e-4)


def _many_antenna_scenario(n_tx, n_rx, n_f=2, dims=(10, 8, 6)):
    rng = np.random.default_rng(n_tx * 1000 + n_rx)
    tx = np.c_[rng.uniform(-0.2, 0.2, (n_tx, 2)), np.zeros(n_tx)]
    rx = np.c_[rng.uniform(-0.2, 0.2, (n_rx, 2)), np.zeros(n_rx)]
    return ImagingScenario(array=ArrayGeometry(tuple(map(tuple, tx)), tuple(map(tuple, rx))),
                           frequencies=FrequencyGrid(24e9, 28e9 if n_f > 1 else 24e9, n_f),
                           voxels=VoxelGrid(center=Vec3(0, 0, 0.3), extent=(0.08, 0.06, 0.05), dims=dims))


@pytest.mark.parametrize("n_tx,n_rx", [(150, 150), (8, 300), (40, 260)])
@pytest.mark.parametrize("dtype", DTYPES)
def test_more_than_256_antennas(n_tx, n_rx, dtype, rng):
    """The reference has no antenna cap (geometry.py:50-84): T + R = 300 in both splits, with receivers beyond
    the 8-bit range and up to 75 tx groups, on the flat kernels (forward, adjoint, bit-exact subsets, SPGM
    step) and the separable kernels (a Cartesian batch), against the direct formula."""
    from paper_2509_00774_b200.solver import SPGMEngine

    scn = _many_antenna_scenario(n_tx, n_rx)
    geo = O.geom_from_scenario(scn)
    M = scn.n_channels
    s = rc(rng, scn.n_voxels)
    full = forward_apply(s, scn, dtype=dtype)
    sub = np.sort(rng.choice(M, 3000, replace=False))
    assert rel_l2(full[sub], O.direct_forward(geo, s, sub)) <= TOL[dtype]
    assert np.array_equal(forward_apply(s, scn, subset=sub[::-1], dtype=dtype), full[sub[::-1]])
    r = rc(rng, sub.size)
    assert rel_l2(adjoint_apply(r, scn, subset=sub, dtype=dtype), O.direct_adjoint(geo, r, sub)) <= TOL[dtype]
    # one fused SPGM step
    y = rc(rng, M)
    grad = O.direct_adjoint(geo, O.direct_forward(geo, s, sub) - y[sub], sub) / sub.size
    eta = 0.5 / float(np.max(np.abs(grad)))
    alpha = 0.3 * float(np.median(np.abs(s - eta * grad)))
    plan = DevicePlan(scn, dtype=dtype, structured="never")
    eng = SPGMEngine(plan, y, eta=eta, alpha=alpha, initial=s)
    eng.stage(sub)
    eng.step_staged()
    assert rel_l2(eng.volume(), O.soft_threshold(s - eta * grad, alpha)) <= TOL[dtype]
    # a Cartesian batch on the separable kernels
    fs, ts = np.array([1]), np.sort(rng.choice(n_tx, min(n_tx, 37), replace=False))
    rs = np.sort(rng.choice(n_rx, min(n_rx, 257), replace=False))
    idx = (rs[None, None, :] + n_rx * (ts[None, :, None] + n_tx * fs[:, None, None])).reshape(-1)
    sp = DevicePlan(scn, dtype=dtype, structured="always")
    sp.prepare_structured(fs, ts, rs)
    got = sp.forward(sp._as_dev(s, scn.n_voxels, "s")).to(torch.complex128).cpu().numpy()
    assert rel_l2(got, O.direct_forward(geo, s, idx)) <= TOL[dtype]
    rr = rc(rng, idx.size)
    ga = sp.adjoint(sp._as_dev(rr, idx.size, "r")).to(torch.complex128).cpu().numpy()
    assert rel_l2(ga, O.direct_adjoint(geo, rr, idx)) <= TOL[dtype]


def test_antenna_limits_raise_value_error():
    """Beyond the layout limits the plan refuses with ValueError (no silent truncation)."""
    scn = _many_antenna_scenario(1100, 2, n_f=1, dims=(2, 2, 2))
    with pytest.raises(ValueError, match="transmitters"):
        forward_apply(np.zeros(scn.n_voxels), scn, dtype="c64")



def _tight_scenario():
    """4 + 4 antennas: in c128 the CTA-tile layout leaves no room behind it for staged iterate values (the refilling
    warp loads them into the buffer instead), and the even antenna count takes the bulk-copied D0 row."""
    return ImagingScenario(
        array=ArrayGeometry(((0.03, 0.01, 0.0), (-0.02, 0.04, 0.0), (0.0, -0.05, 0.0), (0.05, 0.05, 0.0)),
                            ((0.01, 0.0, 0.0), (-0.04, -0.01, 0.0), (0.02, -0.03, 0.0), (-0.01, 0.03, 0.0))),
        frequencies=FrequencyGrid(20e9, 30e9, 6),
        voxels=VoxelGrid(center=Vec3(0.0, 0.0, 0.3), extent=(0.2, 0.1, 0.08), dims=(40, 18, 11)),
    )

@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("case", ["medium", "ragged", "small", "tight"])
def test_cta_tile_forward_is_bit_identical(case, dtype, rng, monkeypatch):
    """The CTA-tile forward (fwd_ct_kernel: whole per-tile table resident in shared memory, one CTA per SM over an
    equal range of (tile, channel) pairs) computes every (tile, channel) value with the warp-unit kernel's
    arithmetic and transpose-reduce: forward values must be identical bit for bit (NFGPU_CT=2 forces it whenever
    its layout fits; 0 forbids it), on full sets, subsets and a ragged grid."""
    from paper_2509_00774_b200 import configs
    from paper_2509_00774_b200.forward import forward_values

    if case == "medium":
        scn = configs.medium_scenario()
        idxs = [np.sort(rng.choice(scn.n_channels, 512, replace=False)), np.arange(scn.n_channels)]
    elif case == "small":
        scn = configs.small_scenario()
        idxs = [np.sort(rng.choice(scn.n_channels, 32, replace=False)), np.arange(scn.n_channels)]
    elif case == "tight":
        scn = _tight_scenario()
        idxs = [np.arange(scn.n_channels), np.sort(rng.choice(scn.n_channels, 41, replace=False))]
    else:
        scn = ImagingScenario(
            array=ArrayGeometry(((0.03, 0.01, 0.0), (-0.02, 0.04, 0.0), (0.0, -0.05, 0.0)),
                                ((0.01, 0.0, 0.0), (-0.04, -0.01, 0.0))),
            frequencies=FrequencyGrid(20e9, 30e9, 5),
            voxels=VoxelGrid(center=Vec3(0.0, 0.0, 0.3), extent=(0.2, 0.07, 0.06), dims=(33, 11, 9)),
        )
        idxs = [np.arange(scn.n_channels), np.sort(rng.choice(scn.n_channels, 17, replace=False))]
    s = rc(rng, scn.n_voxels)
    out = {}
    for mode in ("0", "2"):
        monkeypatch.setenv("NFGPU_CT", mode)
        plan = DevicePlan(scn, dtype=dtype, device="cuda:0", structured="never")
        out[mode] = [forward_values(plan, s, idx) for idx in idxs]
    for a, b in zip(out["0"], out["2"]):
        assert np.array_equal(a, b)
    # ... whatever the CTA ranges' cuts (equal ranges, the default piece cost, a large one)
    for cost in ("0", "400"):
        monkeypatch.setenv("NFGPU_CT_COST_FWD", cost)
        plan = DevicePlan(scn, dtype=dtype, device="cuda:0", structured="never")
        for idx, b in zip(idxs, out["2"]):
            assert np.array_equal(forward_values(plan, s, idx), b)


@pytest.mark.parametrize("cost", [None, "0", "400"])
@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("case", ["medium", "ragged", "tight"])
def test_cta_tile_adjoint_prox_matches_warp_unit(case, dtype, cost, rng, monkeypatch):
    """The CTA-tile adjoint + prox (adj_ct_kernel: warps split each piece's channels, the last one sums their
    partial gradients in warp order, the pieces' epilogues run side by side at the end; tiles cut across CTAs sum
    their pieces in piece order) against the warp-unit kernel: the same SPGM step to rounding, and the
    statistics too (NFGPU_CT=2 forces the CTA-tile kernels whenever the layout fits, NFGPU_CT_ADJ=0 keeps the
    adjoint on the warp-unit kernel)."""
    from paper_2509_00774_b200 import configs
    from paper_2509_00774_b200.solver import SPGMEngine

    if cost is not None:  # the CTA ranges' cuts (ct_args): equal ranges, or a large piece cost; default otherwise
        monkeypatch.setenv("NFGPU_CT_COST_ADJ", cost)
    if case == "medium":
        scn = configs.medium_scenario()
        B = 512
    elif case == "tight":
        scn = _tight_scenario()
        B = 57
    else:
        scn = ImagingScenario(
            array=ArrayGeometry(((0.03, 0.01, 0.0), (-0.02, 0.04, 0.0), (0.0, -0.05, 0.0)),
                                ((0.01, 0.0, 0.0), (-0.04, -0.01, 0.0))),
            frequencies=FrequencyGrid(20e9, 30e9, 5),
            voxels=VoxelGrid(center=Vec3(0.0, 0.0, 0.3), extent=(0.2, 0.07, 0.06), dims=(33, 11, 9)),
        )
        B = 23
    s = rc(rng, scn.n_voxels)
    y = rc(rng, scn.n_channels)
    idx = np.sort(rng.choice(scn.n_channels, B, replace=False))
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("NFGPU_CT", "2")
        monkeypatch.setenv("NFGPU_CT_ADJ", mode)
        plan = DevicePlan(scn, dtype=dtype, device="cuda:0", structured="never")
        eng = SPGMEngine(plan, y, eta=2e-3, alpha=0.05, initial=s)
        eng.stage(idx)
        eng.step_staged()
        out[mode] = (eng.volume(), eng.stats.cpu().numpy())
    tol = 1e-5 if dtype == "c64" else 1e-12
    assert rel_l2(out["1"][0], out["0"][0]) <= tol
    np.testing.assert_allclose(out["1"][1], out["0"][1], rtol=tol)
