"""Oracle parity for the BASELINE configs the reference cannot run itself (its phasor tables
would need 206 GB at Large and 137 GB-1.9 TB for the microbenchmark):

* config 4, the operator microbenchmark, on all three grids (64³ in test_gpu_operator.py,
  128³ and 192x192x96 here), c64 and c128, flat and separable kernels: sampled output rows
  (forward) and sampled voxels (adjoint) against the oracle's direct formula
  (oracle/nfmimo_oracle.py direct_forward / direct_adjoint, a restatement of forward.py:142-155);
* config 3, the minibatch sweep: one SPGM step at |B| in {256, 16384, 65536} on the flat kernels
  and one ISTA step (|B| = M) on the structured / tcgen05 route, on a Large sub-slab;
* a c128 Large spot check, which pins the c128 path that serves as the proxy oracle of the
  500-iteration Large test (test_gpu_solver.py).

Tolerances (north star): c64 <= 1e-5, c128 <= 1e-10 relative L2.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import rc, rel_l2
from oracle import nfmimo_oracle as O
from paper_2509_00774_b200 import adjoint_apply, configs, forward_apply
from paper_2509_00774_b200.plan import DevicePlan
from paper_2509_00774_b200.solver import SPGMEngine

pytestmark = pytest.mark.gpu
TOL = {"c128": 1e-10, "c64": 1e-5}
DTYPES = ("c128", "c64")


def _adjoint_at(geo, r, idx, vox, step=131072):
    return sum(O.direct_adjoint(geo, r[a:a + step], idx[a:a + step], voxels=vox) for a in range(0, idx.size, step))


@pytest.mark.parametrize("structured", [False, True])
@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("grid", ["128^3", "192x192x96"])
def test_microbenchmark_grids_spot_check(grid, dtype, structured):
    """One full-M forward and one full-M adjoint (M = 64 x 64 x 256 = 1,048,576) with N(0,1) complex
    inputs, checked at 12 rows and 8 voxels against the direct formula."""
    scn = configs.micro_scenario(grid)
    geo = O.geom_from_scenario(scn)
    rng = np.random.default_rng(13)
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
    rows = np.sort(rng.choice(scn.n_channels, 12, replace=False))
    assert rel_l2(y[rows], O.direct_forward(geo, s, rows, chunk=32768)) <= TOL[dtype]
    g = plan.adjoint(plan._as_dev(r, scn.n_channels, "r")).to(torch.complex128).cpu().numpy()
    vox = np.sort(rng.choice(scn.n_voxels, 8, replace=False))
    assert rel_l2(g[vox], _adjoint_at(geo, r, np.arange(scn.n_channels), vox)) <= TOL[dtype]
    del plan
    torch.cuda.empty_cache()


def test_large_c128_spot_check():
    """The c128 path on the full Large grid (the proxy oracle of the 500-iteration Large test)."""
    scn = configs.large_scenario()
    geo = O.geom_from_scenario(scn)
    rng = np.random.default_rng(6)
    s = rc(rng, scn.n_voxels)
    idx = np.sort(rng.choice(scn.n_channels, 4096, replace=False))
    y = forward_apply(s, scn, subset=idx, dtype="c128")
    rows = rng.choice(idx.size, 16, replace=False)
    assert rel_l2(y[rows], O.direct_forward(geo, s, idx[rows], chunk=65536)) <= 1e-10
    r = rc(rng, idx.size)
    g = adjoint_apply(r, scn, subset=idx, dtype="c128")
    vox = rng.choice(scn.n_voxels, 1024, replace=False)
    assert rel_l2(g[vox], O.direct_adjoint(geo, r, idx, voxels=vox)) <= 1e-10


def _slab_step_check(plan, geo, idx, dtype, rng, structured=False):
    """One fused SPGM step on ``plan`` (a Large sub-slab) against the oracle: forward rows and adjoint
    voxels by the direct formula, then the step s+ = soft(s - eta/B A^H(A s - y), alpha) at sampled
    voxels, with A s taken from the c128 path whose rows were just pinned."""
    n = plan.n_local
    s = rc(rng, n)
    y = rc(rng, geo.M) * 1e-3
    B = idx.size
    if structured:
        assert plan.try_structured(idx)
    else:
        plan.prepare(torch.from_numpy(idx.astype(np.int32)).to(plan.device))
    sd = plan._as_dev(s, n, "s")
    yb = plan.forward(sd).to(torch.complex128).cpu().numpy()
    rows = np.sort(rng.choice(B, 12, replace=False))
    assert rel_l2(yb[rows], O.direct_forward(geo, s, idx[rows], chunk=16384)) <= TOL[dtype]
    ref128 = DevicePlan(plan.scenario, dtype="c128", z_range=plan.z_range, max_batch=B, structured="never")
    ref128.prepare(torch.from_numpy(idx.astype(np.int32)).to(ref128.device))
    y128 = ref128.forward(ref128._as_dev(s, n, "s")).cpu().numpy()
    assert rel_l2(y128[rows], O.direct_forward(geo, s, idx[rows], chunk=16384)) <= 1e-10
    del ref128
    resid = y128 - y[idx]
    vox = np.sort(rng.choice(n, 64, replace=False))
    grad = _adjoint_at(geo, resid, idx, vox) / B
    eta = 0.5 / float(np.max(np.abs(grad)))
    alpha = 0.3 * float(np.median(np.abs(s[vox] - eta * grad)))
    eng = SPGMEngine(plan, y, eta=eta, alpha=alpha, initial=s)
    if structured:
        eng.stage(idx)
        assert plan.staged_structured
    else:
        eng.stage(torch.from_numpy(idx.astype(np.int32)).to(plan.device))
    eng.step_staged()
    got = eng.volume()[vox]
    ref = O.soft_threshold(s[vox] - eta * grad, alpha)
    assert np.count_nonzero(ref) not in (0, ref.size)
    assert rel_l2(got, ref) <= TOL[dtype]


@pytest.mark.parametrize("batch", [256, 16384, 65536])
def test_sweep_spgm_step_on_large_slab(batch):
    """BASELINE config 3 (minibatch sweep on the Large geometry), c64 flat kernels, one SPGM step."""
    scn = configs.large_scenario()
    z = (20, 24)
    geo = O.geom_from_scenario(scn, z_range=z)
    rng = np.random.default_rng(batch)
    idx = np.sort(rng.choice(scn.n_channels, batch, replace=False))
    plan = DevicePlan(scn, dtype="c64", z_range=z, max_batch=batch, structured="never")
    _slab_step_check(plan, geo, idx, "c64", rng)


def test_sweep_ista_step_on_large_slab_structured():
    """The sweep's deterministic reference (ISTA, |B| = M = 294,912) on the separable route: the full
    set is Cartesian, so the step runs on the tcgen05 adjoint (+ prox) and the structured forward."""
    scn = configs.large_scenario()
    z = (20, 24)
    geo = O.geom_from_scenario(scn, z_range=z)
    rng = np.random.default_rng(99)
    idx = np.arange(scn.n_channels)
    plan = DevicePlan(scn, dtype="c64", z_range=z, structured="auto")
    _slab_step_check(plan, geo, idx, "c64", rng, structured=True)
