"""The fused peer all-reduce of the forward partials (nf_comm_*) on one B200.

Real multi-GPU runs need several GPUs, and ranks whose kernels wait on one another must not run as
separate launches on one GPU. So the protocol (per-rank pushes into every rank's slots, release/
acquire flags per (source rank, block), epoch counters, parity double-buffering, fixed rank order)
is exercised by nf_comm_emulate: `world` ranks emulated in ONE cooperative launch, every block
co-resident. The production entry point (nf_forward_allreduce, SPGMEngine(collective="peer")) is
run at world size 1, where it must reproduce the plain forward and SPGM iterates bit for bit."""

from __future__ import annotations

import ctypes
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _emulate(dtype: int, world: int, span: int, nseg: int, epochs: int, seed: int = 0):
    from paper_2509_00774_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(seed)
    n_f = 7
    tmp = rng.standard_normal((epochs, world, max(nseg, 1), span, 2))
    sf = rng.integers(0, n_f, span).astype(np.int32)
    spos = rng.permutation(span).astype(np.int32)
    pulse = rng.standard_normal((n_f, 2))
    y = np.zeros((epochs, world, span, 2))
    dp = ctypes.POINTER(ctypes.c_double)
    ip = ctypes.POINTER(ctypes.c_int)
    rc = lib.nf_comm_emulate(dtype, world, span, nseg, epochs, tmp.ctypes.data_as(dp), sf.ctypes.data_as(ip),
                             spos.ctypes.data_as(ip), pulse.ctypes.data_as(dp), n_f, y.ctypes.data_as(dp))
    _lib.check(rc, "nf_comm_emulate")
    if nseg == 0:  # one-shot variant: each rank's input is its finished y (as stored in Real)
        yin = tmp[:, :, 0].astype(np.float32 if dtype == _lib.NF_C64 else np.float64).astype(np.float64)
        tot = np.zeros((epochs, span, 2))
        for q in range(world):
            tot += yin[:, q]
        return y[..., 0] + 1j * y[..., 1], tot[..., 0] + 1j * tot[..., 1]
    # expected: per rank, segments summed in order; then ranks summed in order; times p_f/(4π)
    part = np.zeros((epochs, world, span, 2))
    for s in range(nseg):
        part += tmp[:, :, s]
    tot = np.zeros((epochs, span, 2))
    for q in range(world):
        tot += part[:, q]
    p = (pulse[sf, 0] + 1j * pulse[sf, 1]) / (4 * np.pi)
    val = p * (tot[..., 0] + 1j * tot[..., 1])
    exp = np.zeros((epochs, span), complex)
    exp[:, spos] = val
    got = y[..., 0] + 1j * y[..., 1]
    return got, exp


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_emulated_ranks_c128(world):
    from paper_2509_00774_b200 import _lib

    got, exp = _emulate(_lib.NF_C128, world, span=1000, nseg=5, epochs=5)
    for q in range(world):  # every rank holds the same bits
        assert np.array_equal(got[:, q], got[:, 0])
    err = np.linalg.norm(got[:, 0] - exp) / np.linalg.norm(exp)
    assert err <= 1e-15, err


def test_emulated_ranks_c64_many_epochs():
    from paper_2509_00774_b200 import _lib

    # 11 epochs: both parities of the receive slots are reused several times
    got, exp = _emulate(_lib.NF_C64, 4, span=4096, nseg=3, epochs=11, seed=1)
    for q in range(4):
        assert np.array_equal(got[:, q], got[:, 0])
    err = np.linalg.norm(got[:, 0] - exp) / np.linalg.norm(exp)
    assert err <= 1e-7, err


@pytest.mark.parametrize("world", [2, 5])
def test_emulated_ranks_one_shot(world):
    from paper_2509_00774_b200 import _lib

    for dt, tol in ((_lib.NF_C128, 1e-15), (_lib.NF_C64, 1e-7)):
        got, exp = _emulate(dt, world, span=777, nseg=0, epochs=4, seed=world)
        for q in range(world):
            assert np.array_equal(got[:, q], got[:, 0])
        err = np.linalg.norm(got[:, 0] - exp) / np.linalg.norm(exp)
        assert err <= tol, (dt, err)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("structured", [False, True])
def test_forward_allreduce_world1_bitwise(structured):
    from paper_2509_00774_b200 import configs
    from paper_2509_00774_b200.plan import DevicePlan

    scn = configs.medium_scenario()
    plan = DevicePlan(scn, dtype="c64", device="cuda:0", max_batch=4096)
    h = plan.comm_create(0, 1)
    assert len(h) == 64
    plan.comm_connect([h])
    rng = np.random.default_rng(3)
    s = plan._as_dev(rng.standard_normal(scn.n_voxels) + 1j * rng.standard_normal(scn.n_voxels), scn.n_voxels, "s")
    if structured:
        plan.prepare_structured(np.array([1, 5, 9]), np.arange(16), np.arange(16))
    else:
        idx = np.sort(rng.choice(scn.n_channels, 2000, replace=False))
        plan.prepare(torch.from_numpy(idx.astype(np.int32)).cuda())
    for _ in range(3):  # several epochs
        a = plan.forward(s)
        b = plan.forward_allreduce(s)
        torch.cuda.synchronize()
        assert torch.equal(a, b)
    assert not plan.comm_timed_out()


def test_spgm_engine_peer_world1_matches_unsharded():
    import torch.distributed as dist

    from paper_2509_00774_b200 import configs
    from paper_2509_00774_b200.plan import DevicePlan
    from paper_2509_00774_b200.solver import SPGMEngine

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        scn = configs.medium_scenario()
        rng = np.random.default_rng(5)
        y = rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)
        p1 = DevicePlan(scn, dtype="c64", device="cuda:0", max_batch=512)
        p2 = DevicePlan(scn, dtype="c64", device="cuda:0", max_batch=512)
        e1 = SPGMEngine(p1, y, 1e-2, 1e-6)
        e2 = SPGMEngine(p2, y, 1e-2, 1e-6, process_group=dist.group.WORLD, collective="peer")
        assert e2.collective == "peer"
        for k in range(4):
            e1.sample_device(7, k, 512)
            e2.sample_device(7, k, 512)
            e1.step_staged()
            e2.step_staged()
        g = e2.graph(7, 512, pairs=1)  # the peer kernel inside a CUDA graph
        g1 = e1.graph(7, 512, pairs=1)
        g.replay()
        g1.replay()
        torch.cuda.synchronize()
        assert torch.equal(e1.s, e2.s)
        assert e2.magnitude_change() == e1.magnitude_change()
    finally:
        dist.destroy_process_group()


def test_forward_allreduce_world1_multiwindow_flat():
    """Large, a flat batch of 40,000 channels: three forward windows (16,384-channel partial buffer),
    each fused with the peer all-reduce at its 256-aligned channel offset."""
    from paper_2509_00774_b200 import configs
    from paper_2509_00774_b200.plan import DevicePlan

    scn = configs.WORKLOADS["large"]().scenario
    plan = DevicePlan(scn, dtype="c64", device="cuda:0", max_batch=40000, structured="never")
    plan.comm_connect([plan.comm_create(0, 1)])
    rng = np.random.default_rng(9)
    s = plan._as_dev(rng.standard_normal(scn.n_voxels) + 1j * rng.standard_normal(scn.n_voxels), scn.n_voxels, "s")
    idx = np.sort(rng.choice(scn.n_channels, 40000, replace=False))
    plan.prepare(torch.from_numpy(idx.astype(np.int32)).cuda())
    for _ in range(2):
        a = plan.forward(s)
        b = plan.forward_allreduce(s)
        torch.cuda.synchronize()
        assert torch.equal(a, b)
    assert not plan.comm_timed_out()
