"""GPU parity of the structured (Cartesian) fast path, nf_batch_prepare_structured.

A structured batch Fs × Ts × Rs is what the reference's sample_minibatch draws
(pkg/src/nfmimo/solver.py:205-225) and what the full channel set is. The separable kernels
must give the same operator as the flat path: the oracle's direct formula (relative L2
≤ 1e-10 in complex128, ≤ 1e-5 in complex64), the flat path on the same channel list, and
the reference's structured-SPGM fixture."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden, rc, rel_l2, small
from oracle import nfmimo_oracle as O
from paper_2509_00774_b200 import (
    ArrayGeometry,
    FrequencyGrid,
    ImagingScenario,
    MinibatchComposition,
    SolverConfig,
    Vec3,
    VoxelGrid,
    configs,
    spgm_solve,
)
from paper_2509_00774_b200.forward import get_plan
from paper_2509_00774_b200.plan import DevicePlan, cartesian_factors

pytestmark = pytest.mark.gpu
TOL = {"c128": 1e-10, "c64": 1e-5}
DTYPES = ("c128", "c64")


def product_indices(fs, ts, rs, T, R):
    fs, ts, rs = (np.asarray(a, dtype=np.int64) for a in (fs, ts, rs))
    return (rs[None, None, :] + R * (ts[None, :, None] + T * fs[:, None, None])).reshape(-1)


def ragged_scenario(n_tx=5, n_rx=11, n_f=4, dims=(13, 6, 5)):
    """Odd transmitter count, receivers not a multiple of the 8-receiver staging block,
    voxel dims not multiples of the 8×8×4 warp tile."""
    rng = np.random.default_rng(77)
    tx = tuple(Vec3(*p) for p in np.c_[rng.uniform(-0.1, 0.1, (n_tx, 2)), np.zeros(n_tx)])
    rx = tuple(Vec3(*p) for p in np.c_[rng.uniform(-0.1, 0.1, (n_rx, 2)), np.zeros(n_rx)])
    return ImagingScenario(array=ArrayGeometry(tx, rx), frequencies=FrequencyGrid(57e9, 64e9, n_f),
                           voxels=VoxelGrid(center=Vec3(0, 0, 0.35), extent=(0.1, 0.06, 0.05), dims=dims))


@pytest.fixture(params=["ffma", "tc"])
def adj_kernel(request, monkeypatch):
    """Structured c64 adjoint on the FFMA kernel (NFGPU_TC=0) or forced onto the tcgen05 kernel
    (NFGPU_TC=2, whatever the batch shape); read at plan creation."""
    monkeypatch.setenv("NFGPU_TC", "0" if request.param == "ffma" else "2")
    return request.param


def adjoint_launches(plan, r):
    """Kernel launches of one plain adjoint: 2 on the FFMA path, 3 on the tensor-core path (B prep)."""
    n0 = plan.info()["launches"]
    plan.adjoint(r)
    return plan.info()["launches"] - n0


def draw(rng, n, k):
    return np.sort(rng.choice(n, size=k, replace=False)).astype(np.int32)


def run_both(plan, s, r, fs, ts, rs):
    plan.prepare_structured(fs, ts, rs)
    y = plan.forward(plan._as_dev(s, plan.n_local, "s"))
    g = plan.adjoint(plan._as_dev(r, plan.B, "r"))
    return y.to(torch.complex128).cpu().numpy(), g.to(torch.complex128).cpu().numpy()


def test_cartesian_detection():
    T, R = 5, 7
    idx = product_indices([0, 2], [1, 3, 4], [0, 6], T, R)
    fs, ts, rs = cartesian_factors(idx, T, R)
    assert fs.tolist() == [0, 2] and ts.tolist() == [1, 3, 4] and rs.tolist() == [0, 6]
    assert cartesian_factors(idx[::-1], T, R) is None  # not in sorted order
    assert cartesian_factors(idx[:-1], T, R) is None  # not a full product
    assert cartesian_factors(np.array([3]), T, R) is not None  # one channel is a 1×1×1 product


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("builder", [small, ragged_scenario], ids=["small", "ragged"])
def test_structured_matches_oracle(builder, dtype, adj_kernel):
    if dtype == "c128" and adj_kernel == "tc":
        pytest.skip("the tensor-core adjoint is c64 only")
    scn = builder()
    plan = DevicePlan(scn, dtype=dtype)
    g = O.geom_from_scenario(scn)
    rng = np.random.default_rng(5)
    T, R, F = scn.array.n_tx, scn.array.n_rx, scn.frequencies.count
    comps = [(F, T, R), (1, 1, 1), (1, T, 1), (F, 1, R), (max(1, F // 2), max(1, T - 1), max(1, R - 2))]
    for kf, kt, kr in comps:
        fs, ts, rs = draw(rng, F, kf), draw(rng, T, kt), draw(rng, R, kr)
        idx = product_indices(fs, ts, rs, T, R)
        s, r = rc(rng, scn.n_voxels), rc(rng, idx.size)
        y, gg = run_both(plan, s, r, fs, ts, rs)
        assert rel_l2(y, O.direct_forward(g, s, idx)) <= TOL[dtype], (kf, kt, kr)
        assert rel_l2(gg, O.direct_adjoint(g, r, idx)) <= TOL[dtype], (kf, kt, kr)


@pytest.mark.parametrize("dtype", DTYPES)
def test_structured_equals_flat_on_medium_full_set(dtype):
    """All M channels of BASELINE Medium: separable vs flat kernels on the same channel list."""
    scn = configs.medium_scenario()
    plan = DevicePlan(scn, dtype=dtype)
    rng = np.random.default_rng(3)
    M = scn.n_channels
    s = plan._as_dev(rc(rng, scn.n_voxels), plan.n_local, "s")
    r = plan._as_dev(rc(rng, M), M, "r")
    plan.prepare(torch.arange(M, dtype=torch.int32, device=plan.device))
    y0, g0 = plan.forward(s).clone(), plan.adjoint(r).clone()
    plan.prepare_full()
    assert plan.staged_structured
    y1, g1 = plan.forward(s), plan.adjoint(r)
    tol = {"c128": 1e-11, "c64": 1e-5}[dtype]
    to = lambda t: t.to(torch.complex128).cpu().numpy()  # noqa: E731
    assert rel_l2(to(y1), to(y0)) <= tol
    assert rel_l2(to(g1), to(g0)) <= tol


@pytest.mark.parametrize("dtype", DTYPES)
def test_structured_adjoint_prox_equals_flat(dtype, adj_kernel):
    if dtype == "c128" and adj_kernel == "tc":
        pytest.skip("the tensor-core adjoint is c64 only")
    scn = configs.medium_scenario()
    plan = DevicePlan(scn, dtype=dtype)
    rng = np.random.default_rng(8)
    T, R, F = scn.array.n_tx, scn.array.n_rx, scn.frequencies.count
    fs, ts, rs = draw(rng, F, 8), draw(rng, T, 9), draw(rng, R, 12)
    idx = product_indices(fs, ts, rs, T, R)
    B = idx.size
    s_in = plan._as_dev(rc(rng, scn.n_voxels) * 1e-3, plan.n_local, "s")
    r = plan._as_dev(rc(rng, B), B, "r")
    y = plan._as_dev(rc(rng, plan.M), plan.M, "y")
    outs = []
    for structured in (False, True):
        if structured:
            plan.prepare_structured(fs, ts, rs)
        else:
            plan.prepare(torch.from_numpy(idx.astype(np.int32)).to(plan.device))
        s_out = torch.empty_like(s_in)
        st = torch.zeros(4, dtype=torch.float64, device=plan.device)
        plan.adjoint_prox(r, y, s_in, s_out, 0.5 / B, 1e-6, st)
        outs.append((s_out.to(torch.complex128).cpu().numpy(), st.cpu().numpy()))
    tol = {"c128": 1e-11, "c64": 1e-5}[dtype]
    assert rel_l2(outs[1][0], outs[0][0]) <= tol
    assert np.allclose(outs[1][1], outs[0][1], rtol=tol * 10)
    if dtype == "c64":
        assert adjoint_launches(plan, r) == (3 if adj_kernel == "tc" else 2)
    # ½‖r − y_B‖²: same terms, summed in each path's own sorted order
    assert outs[1][1][2] == pytest.approx(outs[0][1][2], rel=1e-12)


def test_structured_slab_plans_sum_to_full():
    scn = configs.medium_scenario()
    rng = np.random.default_rng(4)
    s, r = rc(rng, scn.n_voxels), rc(rng, scn.n_channels)
    full = DevicePlan(scn, dtype="c128")
    full.prepare_full()
    y_full = full.forward(full._as_dev(s, full.n_local, "s")).cpu().numpy()
    g_full = full.adjoint(full._as_dev(r, full.M, "r")).cpu().numpy()
    nz = scn.voxels.dims[2]
    y_sum = np.zeros_like(y_full)
    g_cat = []
    for z0, z1 in [(0, 5), (5, 17), (17, nz)]:
        p = DevicePlan(scn, dtype="c128", z_range=(z0, z1))
        p.prepare_full()
        y_sum += p.forward(p._as_dev(s[p.vox_offset:p.vox_offset + p.n_local], p.n_local, "s")).cpu().numpy()
        g_cat.append(p.adjoint(p._as_dev(r, p.M, "r")).cpu().numpy())
    assert rel_l2(y_sum, y_full) <= 1e-12
    # voxel-local; the chunk count (summation order over channels) follows the slab's tile count
    assert rel_l2(np.concatenate(g_cat), g_full) <= 1e-12


@pytest.mark.parametrize("comp", [(3, 48, 48), (2, 24, 40), (5, 7, 33), (2, 64, 64)])
def test_tensor_core_shapes(comp, monkeypatch):
    """The tcgen05 forward and adjoint (forced) on Large sub-slabs: several K chunks, padded M/N
    (2·n_t, n_r not multiples of 16), receivers not a multiple of the 8-receiver step, against the
    direct formula."""
    monkeypatch.setenv("NFGPU_TC", "2")
    # 64 + 64 antennas (the microbenchmark array): the table leaves room for two pipeline stages only
    scn = configs.micro_scenario("64^3") if comp[1] > 48 else configs.large_scenario()
    z = (20, 24)
    plan = DevicePlan(scn, dtype="c64", z_range=z)
    g = O.geom_from_scenario(scn, z_range=z)
    rng = np.random.default_rng(sum(comp))
    T, R, F = scn.array.n_tx, scn.array.n_rx, scn.frequencies.count
    fs, ts, rs = draw(rng, F, comp[0]), draw(rng, T, comp[1]), draw(rng, R, comp[2])
    idx = product_indices(fs, ts, rs, T, R)
    r = rc(rng, idx.size)
    plan.prepare_structured(fs, ts, rs)
    rd = plan._as_dev(r, plan.B, "r")
    assert adjoint_launches(plan, rd) == 3
    gg = plan.adjoint(rd).to(torch.complex128).cpu().numpy()
    vox = rng.choice(plan.n_local, 96, replace=False)
    assert rel_l2(gg[vox], O.direct_adjoint(g, r, idx, voxels=vox)) <= 1e-5
    s = rc(rng, plan.n_local)
    y = plan.forward(plan._as_dev(s, plan.n_local, "s")).to(torch.complex128).cpu().numpy()
    assert rel_l2(y, O.direct_forward(g, s, idx)) <= 1e-5


def test_structured_large_window_chunking():
    """Large (M = 294,912): the full set needs many forward launch windows; check a window
    boundary row and the adjoint on a sub-slab against the direct formula."""
    scn = configs.large_scenario()
    z = (30, 34)
    plan = DevicePlan(scn, dtype="c64", z_range=z)
    g = O.geom_from_scenario(scn, z_range=z)
    rng = np.random.default_rng(6)
    s = rc(rng, plan.n_local)
    plan.prepare_full()
    y = plan.forward(plan._as_dev(s, plan.n_local, "s")).to(torch.complex128).cpu().numpy()
    # the forward window holds fwd_chunk // n_rx whole (f, t) rows (nfgpu.cu launch_forward_struct)
    fwd_chunk = max(1024, min(plan.M, (512 << 20) // (plan.info()["tiles"] * 2 * 4)))
    edge = (fwd_chunk // scn.array.n_rx) * scn.array.n_rx
    assert edge < plan.M
    pick = np.unique(np.r_[rng.choice(plan.M, 200, replace=False), 0, plan.M - 1, np.arange(edge - 40, edge + 40)])
    assert rel_l2(y[pick], O.direct_forward(g, s, pick)) <= 1e-5
    r = rc(rng, plan.M)
    gg = plan.adjoint(plan._as_dev(r, plan.M, "r")).to(torch.complex128).cpu().numpy()
    vox = rng.choice(plan.n_local, 64, replace=False)
    ref = sum(O.direct_adjoint(g, r[a:a + 65536], np.arange(a, min(a + 65536, plan.M)), voxels=vox)
              for a in range(0, plan.M, 65536))
    assert rel_l2(gg[vox], ref) <= 1e-5


def test_structured_validation(small_scenario):
    plan = DevicePlan(small_scenario, dtype="c64", max_batch=8)
    T, R, F = small_scenario.array.n_tx, small_scenario.array.n_rx, small_scenario.frequencies.count
    with pytest.raises(ValueError, match="increasing"):
        plan.prepare_structured([1, 0], [0], [0])
    with pytest.raises(ValueError, match="increasing"):
        plan.prepare_structured([0], [0, 0], [0])
    with pytest.raises(ValueError, match="out of range"):
        plan.prepare_structured([0], [T], [0])
    with pytest.raises(ValueError, match="out of range"):
        plan.prepare_structured([-1], [0], [0])
    with pytest.raises(ValueError, match="count"):
        plan.prepare_structured([], [0], [0])
    with pytest.raises(ValueError, match="max_batch"):
        plan.prepare_structured(np.arange(F), np.arange(T), np.arange(R))


def test_structured_spgm_matches_reference_fixture_and_flat():
    """The reference's structured SPGM fixture with a composition large enough for the separable
    path (auto policy), and the same run forced onto the flat path."""
    scn = small()
    g = golden("unit_scenarios")
    comp = MinibatchComposition(2, 2, 1)
    plan = get_plan(scn, "c128")
    old = plan.structured
    try:
        plan.structured = "always"
        rep = spgm_solve(g["small_y"], scn, SolverConfig(max_iters=30, tol=1e-300, composition=comp, rng_seed=9))
        assert rel_l2(rep.volume.values, g["small_spgm_structured"]) <= 1e-10
        assert np.allclose([r.magnitude_change for r in rep.per_iteration], g["small_spgm_changes"], rtol=1e-8)
        rng = np.random.default_rng(0)
        y = rc(rng, scn.n_channels)
        cfg = SolverConfig(max_iters=20, tol=1e-300, composition=MinibatchComposition(2, 3, 2), rng_seed=2)
        a = spgm_solve(y, scn, cfg).volume.values
        plan.structured = "never"
        b = spgm_solve(y, scn, cfg).volume.values
        assert rel_l2(a, b) <= 1e-11
    finally:
        plan.structured = old
