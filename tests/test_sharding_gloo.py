"""CPU, world_size 2 over gloo: the voxel-slab sharding used by the multi-GPU path
(paper_2509_00774_b200/sharding.py) reproduces the unsharded operator and
SPGM step. Forward partials over z-slabs are summed by one all-reduce; the adjoint and
prox are slab-local. The oracle stands in for the per-rank kernels here."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import nfmimo_oracle as O
from paper_2509_00774_b200 import configs
from paper_2509_00774_b200.sharding import slab_range


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _allreduce_complex(x: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(torch.view_as_real(t))
    return t.numpy()


def _worker(rank: int, world: int, port: int, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scn = configs.small_scenario()
        nx, ny, nz = scn.voxels.dims
        z0, z1 = slab_range(nz, rank, world)
        geo = O.geom_from_scenario(scn, z_range=(z0, z1))
        rng = np.random.default_rng(0)  # identical on every rank
        s = rng.standard_normal(scn.n_voxels) + 1j * rng.standard_normal(scn.n_voxels)
        y = rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)
        idx = np.sort(rng.choice(scn.n_channels, 32, replace=False))
        lo, hi = nx * ny * z0, nx * ny * z1
        # forward: slab partial + all-reduce
        y_b = _allreduce_complex(O.direct_forward(geo, s[lo:hi], idx))
        # adjoint + prox: slab-local
        eta, alpha = 5.0, 1e-4
        g = O.direct_adjoint(geo, y_b - y[idx], idx) / idx.size
        s_next = O.soft_threshold(s[lo:hi] - eta * g, alpha)
        # termination statistics: two scalars all-reduced
        st = torch.tensor([np.sum(np.abs(s[lo:hi]) ** 2),
                           np.sum((np.abs(s_next) - np.abs(s[lo:hi])) ** 2)], dtype=torch.float64)
        dist.all_reduce(st)
        q.put((rank, (z0, z1), y_b, s_next, st.numpy()))
    finally:
        dist.destroy_process_group()


def test_slab_ranges_partition_planes():
    for nz in (1, 4, 7, 8, 32, 64):
        for world in range(1, min(nz, 8) + 1):
            r = [slab_range(nz, k, world) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == nz
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            assert all(hi > lo for lo, hi in r)
            if nz % 4 == 0 and nz // 4 >= world:
                assert all(lo % 4 == 0 for lo, _ in r)
    with pytest.raises(ValueError):
        slab_range(2, 0, 3)


def test_two_rank_sharded_step_matches_unsharded():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0

    scn = configs.small_scenario()
    geo = O.geom_from_scenario(scn)
    rng = np.random.default_rng(0)
    s = rng.standard_normal(scn.n_voxels) + 1j * rng.standard_normal(scn.n_voxels)
    y = rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)
    idx = np.sort(rng.choice(scn.n_channels, 32, replace=False))
    y_full = O.direct_forward(geo, s, idx)
    g = O.direct_adjoint(geo, y_full - y[idx], idx) / idx.size
    s_next = O.soft_threshold(s - 5.0 * g, 1e-4)
    for _, _, y_b, _, _ in out:  # every rank holds the full reduced forward
        assert np.linalg.norm(y_b - y_full) <= 1e-12 * np.linalg.norm(y_full)
    glued = np.concatenate([o[3] for o in out])
    assert np.linalg.norm(glued - s_next) <= 1e-12 * np.linalg.norm(s_next)
    st = out[0][4]
    change = np.sqrt(st[1]) / max(np.sqrt(st[0]), 1e-12)
    assert change == pytest.approx(O.relative_magnitude_change(s, s_next), rel=1e-10)


def _peer_worker(rank: int, world: int, port: int, q):
    from paper_2509_00774_b200.sharding import connect_peer_allreduce

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = {}

        def create(r, w):  # stands in for nf_comm_create: a rank-specific 64-byte IPC handle
            got["create"] = (r, w)
            return bytes([r + 1]) * 64

        def connect(handles):  # stands in for nf_comm_connect
            got["handles"] = list(handles)

        ok = connect_peer_allreduce(None, dist.group.WORLD, create=create, connect=connect)
        assert ok

        def create_fails_on_1(r, w):  # a rank that cannot export: every rank must learn it, none may hang
            if r == 1:
                raise RuntimeError("no IPC")
            return bytes([r + 1]) * 64

        calls = []
        ok2 = connect_peer_allreduce(None, dist.group.WORLD, create=create_fails_on_1, connect=calls.append)
        q.put((rank, got["create"], got["handles"], ok2, len(calls)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_allreduce_handle_exchange(world):
    """Host side of the fused peer all-reduce (sharding.connect_peer_allreduce): every rank
    exports one handle, and every rank maps the full list in rank order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [bytes([r + 1]) * 64 for r in range(world)]
    for rank, (r, w), handles, ok2, ncalls in out:
        assert (r, w) == (rank, world)
        assert handles == want
        assert ok2 is False and ncalls == 0  # the failure reached every rank, and nobody mapped anything
