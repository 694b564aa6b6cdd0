"""The multi-GPU data path on real kernels: world size 2, both ranks on cuda:0, gloo backend.

Each rank builds a z-slab plan (sharding.slab_range) and runs the sharded SPGMEngine (forward
partial -> all-reduce of 2·|B| reals -> slab-local adjoint + prox) and ShardedSetup (forward_full,
max |A^H y|, power iteration), exactly as bench.py does under torchrun. Gloo's all-reduce is
host-mediated, so no rank's kernels wait on the other's; NCCL needs distinct GPUs and is what the
driver's multi-GPU runs use. Results must match an unsharded run of the same steps."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu
WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(name: str):
    from paper_2509_00774_b200 import configs

    if name == "medium_c64":
        return configs.medium_scenario(), "c64", 512, 1e-5
    return configs.small_scenario(), "c128", 32, 1e-12


def _inputs(scn, B, steps):
    rng = np.random.default_rng(42)  # identical on every rank
    s0 = (rng.standard_normal(scn.n_voxels) + 1j * rng.standard_normal(scn.n_voxels)) * 1e-3
    y = rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)
    idx = [np.sort(rng.choice(scn.n_channels, B, replace=False)) for _ in range(steps)]
    return s0, y, idx


def _run(scn, dtype, s0, y, idx, z_range, pg):
    from paper_2509_00774_b200.plan import DevicePlan
    from paper_2509_00774_b200.sharding import ShardedSetup
    from paper_2509_00774_b200.solver import SPGMEngine

    dev = torch.device("cuda", 0)
    setup = ShardedSetup(scn, dtype=dtype, device=dev, z_range=z_range, process_group=pg)
    y_sim = setup.forward_full(s0 * 1e3)
    amax = setup.max_abs_adjoint(y)
    L = setup.lipschitz(n_iters=6, rng_seed=0)
    plan = DevicePlan(scn, dtype=dtype, device=dev, z_range=z_range, max_batch=max(len(i) for i in idx))
    lo = plan.vox_offset
    eng = SPGMEngine(plan, y, eta=0.5 / L, alpha=1e-6, initial=s0[lo:lo + plan.n_local], process_group=pg)
    changes = []
    for ix in idx:
        eng.stage(ix)
        eng.step_staged()
        changes.append(eng.magnitude_change())
    return {"z": plan.z_range, "vol": eng.volume(), "changes": changes, "y_sim": y_sim, "amax": amax, "L": L}


def _worker(rank, port, name, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_2509_00774_b200.sharding import slab_range

        scn, dtype, B, _ = _case(name)
        s0, y, idx = _inputs(scn, B, steps=4)
        out = _run(scn, dtype, s0, y, idx, slab_range(scn.voxels.dims[2], rank, WORLD), dist.group.WORLD)
        q.put((rank, out))
    except Exception as exc:  # surface worker failures in the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["medium_c64", "small_c128"])
def test_two_rank_slab_sharding_matches_unsharded(name):
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, name, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=120)
    for r, out in results.items():
        assert isinstance(out, dict), f"rank {r}: {out}"
    scn, dtype, B, tol = _case(name)
    s0, y, idx = _inputs(scn, B, steps=4)
    ref = _run(scn, dtype, s0, y, idx, None, None)
    nxy = scn.voxels.dims[0] * scn.voxels.dims[1]
    vol = np.zeros(scn.n_voxels, dtype=complex)
    for r in range(WORLD):
        z0, z1 = results[r]["z"]
        vol[z0 * nxy:z1 * nxy] = results[r]["vol"]
        assert rel_l2(results[r]["y_sim"], ref["y_sim"]) <= tol  # forward partials all-reduced
        assert results[r]["amax"] == pytest.approx(ref["amax"], rel=tol)
        assert results[r]["L"] == pytest.approx(ref["L"], rel=10 * tol)
        assert np.allclose(results[r]["changes"], ref["changes"], rtol=10 * tol)
    assert (results[0]["z"][0], results[1]["z"][1]) == (0, scn.voxels.dims[2])
    assert rel_l2(vol, ref["vol"]) <= tol
