"""GPU parity with a frequency-dependent complex pulse p(f) (TabulatedPulse, reference
geometry.py:239-269) through every kernel that applies it: the flat forward's last reduce
(p_f, forward.py:283-284), the residual records of the adjoint (conj p_f, forward.py:315-325),
the fused adjoint + prox, the structured FFMA and tcgen05 kernels and the world-1 peer
all-reduce. Against the reference's own outputs (tests/golden/pulse_scenarios.npz) and the
oracle's direct formula: c64 <= 1e-5, c128 <= 1e-10 relative L2."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import pulse_cases
from conftest import golden, rc, rel_l2
from oracle import nfmimo_oracle as O
from paper_2509_00774_b200 import (
    MinibatchComposition,
    SolverConfig,
    adjoint_apply,
    forward_apply,
    scenario_fingerprint,
    spgm_solve,
)
from paper_2509_00774_b200.plan import DevicePlan
from paper_2509_00774_b200.solver import SPGMEngine

pytestmark = pytest.mark.gpu
TOL = {"c128": 1e-10, "c64": 1e-5}
DTYPES = ("c128", "c64")
SMALL_CASES = ("tiny", "ragged")


def _pin(name):
    g = golden("pulse_scenarios")
    scn = pulse_cases.CASES[name]()
    assert bytes(g[f"{name}_fingerprint"]) == scenario_fingerprint(scn)
    assert np.iscomplexobj(scn.pulse.evaluate(scn.frequencies.values()))
    return g, scn


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("name", SMALL_CASES)
def test_flat_operator_matches_reference(name, dtype):
    g, scn = _pin(name)
    s, r, sub = g[f"{name}_s"], g[f"{name}_r"], g[f"{name}_sub"]
    tol = TOL[dtype]
    assert rel_l2(forward_apply(s, scn, dtype=dtype), g[f"{name}_fwd"]) <= tol
    assert rel_l2(forward_apply(s, scn, subset=sub, dtype=dtype), g[f"{name}_fwd_sub"]) <= tol
    assert rel_l2(adjoint_apply(r, scn, dtype=dtype), g[f"{name}_adj"]) <= tol
    assert rel_l2(adjoint_apply(r[: sub.size], scn, subset=sub, dtype=dtype), g[f"{name}_adj_sub"]) <= tol


@pytest.mark.parametrize("dtype", DTYPES)
def test_medium_operator_matches_reference(dtype):
    g, scn = _pin("medium")
    idx = g["medium_idx"]
    s = rc(np.random.default_rng(31), scn.n_voxels)  # the generator's draw (make_golden.py gen_pulse)
    assert rel_l2(forward_apply(s, scn, subset=idx, dtype=dtype), g["medium_fwd_sub"]) <= TOL[dtype]
    adj = adjoint_apply(g["medium_r"], scn, subset=idx, dtype=dtype)
    assert rel_l2(adj[g["medium_adj_probe_voxels"]], g["medium_adj_sub_probe"]) <= TOL[dtype]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("name", ("tiny", "ragged", "medium"))
def test_fused_spgm_step_matches_oracle(name, dtype):
    """nf_forward + nf_adjoint_prox (resid records carry conj p_f) against the oracle's step."""
    scn = pulse_cases.CASES[name]()
    geo = O.geom_from_scenario(scn)
    rng = np.random.default_rng(41)
    s, y = rc(rng, scn.n_voxels), rc(rng, scn.n_channels)
    B = min(scn.n_channels, 256)
    idx = np.sort(rng.choice(scn.n_channels, B, replace=False))
    grad = O.direct_adjoint(geo, O.direct_forward(geo, s, idx) - y[idx], idx) / B
    eta = 0.5 / float(np.max(np.abs(grad)))
    alpha = 0.3 * float(np.median(np.abs(s - eta * grad)))
    ref = O.soft_threshold(s - eta * grad, alpha)
    assert np.count_nonzero(ref) not in (0, ref.size)
    plan = DevicePlan(scn, dtype=dtype, device="cuda:0", structured="never")
    eng = SPGMEngine(plan, y, eta=eta, alpha=alpha, initial=s)
    eng.stage(idx)
    eng.step_staged()
    assert rel_l2(eng.volume(), ref) <= TOL[dtype]
    assert eng.magnitude_change() == pytest.approx(O.relative_magnitude_change(s, ref), rel=1e-4)


def _structured_plan(scn, dtype, monkeypatch, kernel):
    monkeypatch.setenv("NFGPU_TC", {"ffma": "0", "tc": "2"}[kernel])
    return DevicePlan(scn, dtype=dtype, device="cuda:0", structured="always")


@pytest.mark.parametrize("kernel,dtype", [("ffma", "c128"), ("ffma", "c64"), ("tc", "c64")])
@pytest.mark.parametrize("name", ("tiny", "ragged", "medium"))
def test_structured_kernels_match_oracle(name, kernel, dtype, monkeypatch):
    """Separable FFMA and tcgen05 kernels (forward, adjoint, adjoint + prox) on Cartesian batches."""
    scn = pulse_cases.CASES[name]()
    geo = O.geom_from_scenario(scn)
    T, R, F = scn.array.n_tx, scn.array.n_rx, scn.frequencies.count
    rng = np.random.default_rng(43)
    fs = np.sort(rng.choice(F, max(1, min(F, 5)), replace=False))
    ts, rs = np.arange(T), np.sort(rng.choice(R, max(1, R - 1), replace=False))
    idx = (rs[None, None, :] + R * (ts[None, :, None] + T * fs[:, None, None])).reshape(-1)
    s, y = rc(rng, scn.n_voxels), rc(rng, scn.n_channels)
    plan = _structured_plan(scn, dtype, monkeypatch, kernel)
    plan.prepare_structured(fs, ts, rs)
    got_f = plan.forward(plan._as_dev(s, scn.n_voxels, "s")).to(torch.complex128).cpu().numpy()
    ref_f = O.direct_forward(geo, s, idx)
    assert rel_l2(got_f, ref_f) <= TOL[dtype]
    r = rc(rng, idx.size)
    got_a = plan.adjoint(plan._as_dev(r, idx.size, "r")).to(torch.complex128).cpu().numpy()
    vox = None if scn.n_voxels <= 4096 else np.sort(rng.choice(scn.n_voxels, 2048, replace=False))
    ref_a = O.direct_adjoint(geo, r, idx, voxels=vox)
    assert rel_l2(got_a if vox is None else got_a[vox], ref_a) <= TOL[dtype]
    # fused adjoint + prox on the same batch
    grad = O.direct_adjoint(geo, ref_f - y[idx], idx, voxels=vox) / idx.size
    s_sel = s if vox is None else s[vox]
    eta = 0.5 / float(np.max(np.abs(grad)))
    alpha = 0.3 * float(np.median(np.abs(s_sel - eta * grad)))
    eng = SPGMEngine(plan, y, eta=eta, alpha=alpha, initial=s)
    eng.stage(idx)
    assert plan.staged_structured
    eng.step_staged()
    got = eng.volume()
    assert rel_l2(got if vox is None else got[vox], O.soft_threshold(s_sel - eta * grad, alpha)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("name", SMALL_CASES)
def test_structured_spgm_matches_reference(name, dtype):
    """Ten structured SPGM iterations (reference sampler, seed 4) against the reference's run."""
    g, scn = _pin(name)
    eta, alpha = (float(v) for v in g[f"{name}_eta_alpha"])
    comp = MinibatchComposition(*(int(v) for v in g[f"{name}_comp"]))
    rep = spgm_solve(g[f"{name}_y"], scn, SolverConfig(eta=eta, alpha=alpha, max_iters=10, tol=1e-300,
                                                       composition=comp, rng_seed=4, dtype=dtype))
    assert rel_l2(rep.volume.values, g[f"{name}_spgm"]) <= (1e-10 if dtype == "c128" else 1e-4)


@pytest.mark.parametrize("structured", [False, True])
@pytest.mark.parametrize("dtype", DTYPES)
def test_forward_allreduce_world1_with_pulse(structured, dtype):
    """The fused peer all-reduce applies p_f after the rank-order sum: at world size 1 it reproduces
    nf_forward bit for bit, and both match the oracle."""
    scn = pulse_cases.medium_pulse()
    geo = O.geom_from_scenario(scn)
    plan = DevicePlan(scn, dtype=dtype, device="cuda:0", max_batch=4096)
    plan.comm_connect([plan.comm_create(0, 1)])
    rng = np.random.default_rng(47)
    s_np = rc(rng, scn.n_voxels)
    s = plan._as_dev(s_np, scn.n_voxels, "s")
    if structured:
        fs, ts, rs = np.array([2, 30, 61]), np.arange(16), np.arange(16)
        plan.prepare_structured(fs, ts, rs)
        idx = (rs[None, None, :] + 16 * (ts[None, :, None] + 16 * fs[:, None, None])).reshape(-1)
    else:
        idx = np.sort(rng.choice(scn.n_channels, 2000, replace=False))
        plan.prepare(torch.from_numpy(idx.astype(np.int32)).cuda())
    for _ in range(2):
        a = plan.forward(s)
        b = plan.forward_allreduce(s)
        torch.cuda.synchronize()
        assert torch.equal(a, b)
    assert not plan.comm_timed_out()
    rows = np.sort(rng.choice(idx.size, 64, replace=False))
    got = b.to(torch.complex128).cpu().numpy()[rows]
    assert rel_l2(got, O.direct_forward(geo, s_np, idx[rows])) <= TOL[dtype]
