"""Voxel-slab sharding across GPUs (one process per GPU, torch.distributed/NCCL).

Rank p owns a contiguous range of z-planes, i.e. the flat voxels
[z0·nx·ny, z1·nx·ny) (x fastest, geometry.py:128-129). Then

    A_B s   = Σ_p A_B[:, slab_p] s[slab_p]    → one all-reduce of 2·|B| reals
    A_B^H r = concat_p A_B[:, slab_p]^H r     → local, no communication
    prox    = per voxel                        → local

Geometry, frequencies and the minibatch are replicated. Every rank derives the same
index list from the same seed, so the index list is never sent. The helpers here also run the setup
computations that need full-M operator applications (measurement simulation,
power-iteration Lipschitz estimate, λ) in the same sharded way.
"""

from __future__ import annotations

import numpy as np
import torch

from .plan import DevicePlan

TILE_Z = 4  # z depth of a warp tile (csrc/nfgpu.cu)


def slab_range(nz: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous z-plane range of ``rank``. Boundaries fall on multiples of the
    tile depth when nz allows it, so no tile straddles two ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if world > nz:
        raise ValueError(f"cannot split {nz} z-planes over {world} ranks")
    unit = TILE_Z if nz % TILE_Z == 0 and nz // TILE_Z >= world else 1
    blocks = nz // unit
    lo = (blocks * rank) // world
    hi = (blocks * (rank + 1)) // world
    return lo * unit, (hi * unit if rank < world - 1 else nz)


def connect_peer_allreduce(plan, process_group, create=None, connect=None) -> bool:
    """Set up the fused peer all-reduce of the forward partials (nf_comm_*) on
    ``plan`` for the ranks of ``process_group``: every rank exports the CUDA IPC handle of its
    receive slots, the handles are all-gathered in rank order over the group (any backend), and
    every rank maps all of them. Every rank runs the same collectives whatever fails locally, and
    the result (True = connected everywhere) is agreed over the group, so no rank can be left
    waiting in a collective the others skipped. Ends with a barrier, so no rank pushes into an
    unmapped peer. ``create``/``connect`` default to the plan's C-ABI calls (tests substitute
    host stand-ins)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(process_group), dist.get_world_size(process_group)
    create = create or plan.comm_create
    connect = connect or plan.comm_connect
    try:
        mine = create(rank, world)
    except Exception:
        mine = None
    handles: list = [None] * world
    dist.all_gather_object(handles, mine, group=process_group)
    ok = mine is not None and all(h is not None for h in handles) and handles[rank] == mine
    if ok:
        try:
            connect(handles)
        except Exception:
            ok = False
    votes: list = [None] * world
    dist.all_gather_object(votes, bool(ok), group=process_group)
    dist.barrier(group=process_group)
    return all(votes)


def peer_allreduce_self_check(plan, process_group, n: int = 1024, rtol: float = 1e-5) -> bool:
    """Start-up check of a connected peer all-reduce on the real ranks: a forward of a fixed random
    iterate over the first min(n, max_batch) channels through nf_forward_allreduce must match nf_forward +
    an all-reduce over the process group (rtol; the two sum in different orders and precisions), with no
    flag wait timing out. Local failures are caught so that every rank runs the same collectives, and the
    verdict is agreed over the group (all ranks pass or all fall back)."""
    import torch.distributed as dist

    dev = plan.device
    B = int(min(n, plan.max_batch, plan.M))
    ok = True
    try:
        gen = torch.Generator(device="cpu").manual_seed(1234)  # the same on every rank
        s = torch.randn(plan.n_local, dtype=plan.torch_dtype, generator=gen).to(dev)
        plan.prepare(torch.arange(B, dtype=torch.int32, device=dev))
        ref = plan.forward(s)
    except Exception:
        ok = False
        ref = torch.zeros(B, dtype=plan.torch_dtype, device=dev)
    dist.all_reduce(torch.view_as_real(ref), group=process_group)
    if ok:
        try:
            got = plan.forward_allreduce(s)
            torch.cuda.synchronize(dev)
            den = torch.clamp(torch.linalg.vector_norm(ref), min=1e-300)
            err = float(torch.linalg.vector_norm(got - ref) / den)
            ok = (not plan.comm_timed_out()) and err <= rtol
        except Exception:
            ok = False
    votes: list = [None] * dist.get_world_size(process_group)
    dist.all_gather_object(votes, bool(ok), group=process_group)
    return all(votes)


def _allreduce(t: torch.Tensor, pg, op=None) -> torch.Tensor:
    if pg is not None:
        if t.is_complex():
            torch.distributed.all_reduce(torch.view_as_real(t), group=pg)
        else:
            torch.distributed.all_reduce(t, op=op or torch.distributed.ReduceOp.SUM, group=pg)
    return t


class ShardedSetup:
    """Full-M operator applications over a slab-sharded plan (setup work, not the hot loop)."""

    def __init__(self, scenario, dtype: str, device, z_range, process_group=None):
        self.scn = scenario
        self.pg = process_group
        self.plan = DevicePlan(scenario, dtype=dtype, device=device, z_range=z_range)
        self.M = scenario.n_channels
        self.plan.prepare_full()

    def _slab(self, x_full: np.ndarray) -> torch.Tensor:
        p = self.plan
        return p._as_dev(np.asarray(x_full)[p.vox_offset:p.vox_offset + p.n_local], p.n_local, "x")

    def forward_full(self, s_full: np.ndarray) -> np.ndarray:
        y = self.plan.forward(self._slab(s_full))
        return _allreduce(y, self.pg).to(torch.complex128).cpu().numpy()

    def max_abs_adjoint(self, y: np.ndarray) -> float:
        g = self.plan.adjoint(self.plan._as_dev(y, self.M, "y"))
        m = g.abs().max().to(torch.float64).reshape(1)
        return float(_allreduce(m, self.pg, torch.distributed.ReduceOp.MAX if self.pg else None).item())

    def lipschitz(self, n_iters: int = 20, rng_seed: int = 0, tol: float = 1e-9) -> float:
        """Power iteration on (1/M) A^H A from the reference's start vector (solver.py:368-397)."""
        n = self.scn.n_voxels
        rng = np.random.default_rng(rng_seed)
        x0 = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        x0 /= np.linalg.norm(x0)
        x = self._slab(x0)
        y = self.plan.vec(self.M)
        z = self.plan.vec(self.plan.n_local)
        lam = 0.0
        for _ in range(n_iters):
            self.plan.forward(x, out=y)
            _allreduce(y, self.pg)
            self.plan.adjoint(y, out=z, scale=1.0 / self.M)
            red = torch.stack([torch.vdot(x, z).real.to(torch.float64),
                               (z.abs().to(torch.float64) ** 2).sum()])
            _allreduce(red, self.pg)
            lam_new, nz = float(red[0]), float(red[1]) ** 0.5
            if nz == 0.0:
                return 0.0
            x = z / nz
            if lam > 0 and abs(lam_new - lam) <= tol * lam:
                return lam_new
            lam = lam_new
        return lam

    def release(self):
        self.plan = None
        torch.cuda.empty_cache()
