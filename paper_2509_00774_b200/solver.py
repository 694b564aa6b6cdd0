"""ℓ1-regularized PGM / SPGM reconstruction — public API of the reference's
``nfmimo.solver`` (pkg/src/nfmimo/solver.py), with the iterate resident on the GPU.

One SPGM iteration (solver.py:281-310) maps to four device steps on one stream:

    sample idx     host numpy, same RNG call sequence as the reference  (solver.py:206-225, 274, 284)
                   or the device Feistel sampler (sampler="device")
    nf_batch_prepare      sort the batch into kernel work order
    nf_forward            y_B = A_B s                                  (solver.py:182)
    nf_adjoint_prox       s⁺ = soft(s − η/B · A_B^H (y_B − y[idx]), α),  plus termination stats
                                                                        (solver.py:183, 288-289)

The only host↔device traffic per iteration is the index list (B int32) and the
four-double stats vector. The stats vector carries the relative magnitude change
the termination test needs (solver.py:302).

Sampling modes (SolverConfig.sampler):
  "host"   (default) composition → structured Cartesian product via the reference
           algorithm; flat_batch → np.sort(rng.choice(M, B, replace=False)).
           Identical index sequence to a reference run with the same seed.
  "device" flat batches drawn on the GPU (keyed Feistel bijection; no host work).
  "table"  an explicit [iters, B] index table (parity runs).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .forward import (
    ChannelSubset,
    MeasurementSet,
    ReflectivityVolume,
    _subset_indices,
    _volume_values,
    adjoint_values,
    default_dtype,
    forward_values,
    get_plan,
)
from .geometry import ImagingScenario
from .plan import DevicePlan, magnitude_change_dev, require_cuda, soft_threshold_dev

__all__ = [
    "MinibatchComposition",
    "SolverConfig",
    "IterationRecord",
    "SolveReport",
    "data_fidelity",
    "full_gradient",
    "minibatch_gradient",
    "sample_minibatch",
    "soft_threshold",
    "relative_magnitude_change",
    "check_termination",
    "pgm_solve",
    "spgm_solve",
    "lipschitz_estimate",
    "SPGMEngine",
]

TERMINATION_TOLERANCE = "tolerance_reached"
TERMINATION_MAX_ITERS = "max_iters"
TERMINATION_TIME_BUDGET = "time_budget"
_ZERO_NORM_GUARD = 1e-12


@dataclass(frozen=True)
class MinibatchComposition:
    """(#frequencies, #transmitters, #receivers) drawn per iteration (solver.py:61-95)."""

    n_f: int
    n_tx: int
    n_rx: int

    def __post_init__(self):
        for k in ("n_f", "n_tx", "n_rx"):
            v = int(getattr(self, k))
            if v < 1:
                raise ValueError(f"{k} must be >= 1, got {v}")
            object.__setattr__(self, k, v)

    @property
    def batch_size(self) -> int:
        return self.n_f * self.n_tx * self.n_rx

    def validate_for(self, scenario: ImagingScenario) -> None:
        caps = (scenario.frequencies.count, scenario.array.n_tx, scenario.array.n_rx)
        for k, v, cap in zip(("n_f", "n_tx", "n_rx"), (self.n_f, self.n_tx, self.n_rx), caps):
            if v > cap:
                raise ValueError(f"{k}={v} exceeds the scenario axis size {cap}")

    def is_full_for(self, scenario: ImagingScenario) -> bool:
        return (self.n_f, self.n_tx, self.n_rx) == (
            scenario.frequencies.count,
            scenario.array.n_tx,
            scenario.array.n_rx,
        )


@dataclass
class SolverConfig:
    """Reference fields (solver.py:98-128) plus the GPU controls.

    dtype       "c128" (default, parity) or "c64" (performance).
    flat_batch  B for flat uniform sampling without replacement (BASELINE configs);
                mutually exclusive with ``composition``.
    sampler     "host" | "device" | "table" (see module docstring).
    index_table [iters, B] int array for sampler="table".
    check_every read the termination stats back every k iterations (1 = reference semantics).
    """

    eta: float = 1e-3
    alpha: float = 4e-5
    max_iters: int = 1000
    tol: float = 1e-3
    rng_seed: int = 0
    composition: MinibatchComposition | None = None
    time_budget_s: float | None = None
    threads: int = 1
    dtype: str | None = None
    flat_batch: int | None = None
    sampler: str = "host"
    index_table: np.ndarray | None = None
    check_every: int = 1

    def __post_init__(self):
        if not (math.isfinite(self.eta) and self.eta > 0):
            raise ValueError(f"eta must be > 0, got {self.eta}")
        if not (math.isfinite(self.alpha) and self.alpha >= 0):
            raise ValueError(f"alpha must be >= 0, got {self.alpha}")
        if int(self.max_iters) < 1:
            raise ValueError(f"max_iters must be >= 1, got {self.max_iters}")
        self.max_iters = int(self.max_iters)
        if not (math.isfinite(self.tol) and self.tol > 0):
            raise ValueError(f"tol must be > 0, got {self.tol}")
        if self.time_budget_s is not None and not self.time_budget_s > 0:
            raise ValueError(f"time_budget_s must be > 0, got {self.time_budget_s}")
        if int(self.threads) < 1:
            raise ValueError("threads must be >= 1")
        if self.sampler not in ("host", "device", "table"):
            raise ValueError(f"sampler must be host/device/table, got {self.sampler!r}")
        if self.flat_batch is not None:
            if int(self.flat_batch) < 1:
                raise ValueError("flat_batch must be >= 1")
            if self.composition is not None:
                raise ValueError("give either composition or flat_batch, not both")
            self.flat_batch = int(self.flat_batch)
        if int(self.check_every) < 1:
            raise ValueError("check_every must be >= 1")
        if self.sampler == "device" and self.composition is None and self.flat_batch is None:
            raise ValueError("sampler='device' needs flat_batch or composition")
        if self.sampler == "table":
            if self.index_table is None:
                raise ValueError("sampler='table' needs index_table")
            if len(self.index_table) < self.max_iters:
                raise ValueError("index_table has fewer rows than max_iters")


@dataclass
class IterationRecord:
    iter: int
    magnitude_change: float
    elapsed_seconds: float
    batch_size: int


@dataclass
class SolveReport:
    volume: ReflectivityVolume
    iterations: int
    wall_time_s: float
    per_iteration: list = field(default_factory=list)
    termination: str = TERMINATION_MAX_ITERS


# ------------------------------------------------------------------ helpers


def _measurement_values(y, scenario: ImagingScenario) -> np.ndarray:
    if isinstance(y, MeasurementSet):
        if not y.matches(scenario):
            raise ValueError(
                "measurement fingerprint does not match the scenario (wrong scenario or stale measurement file)"
            )
        return y.values
    v = np.asarray(y, dtype=np.complex128)
    if v.shape != (scenario.n_channels,):
        raise ValueError(f"expected {scenario.n_channels} measurements, got shape {v.shape}")
    return v


def _subset_or_all(subset, scenario: ImagingScenario) -> np.ndarray:
    if subset is None:
        return np.arange(scenario.n_channels, dtype=np.int64)
    if isinstance(subset, ChannelSubset):
        return subset.indices
    return ChannelSubset(np.asarray(subset)).indices


def _volume_like(s, scenario: ImagingScenario) -> np.ndarray:
    if isinstance(s, ReflectivityVolume):
        if s.grid != scenario.voxels:
            raise ValueError("initial volume grid does not match the scenario")
        return s.values
    v = np.asarray(s, dtype=np.complex128)
    if v.shape != (scenario.n_voxels,):
        raise ValueError(f"expected {scenario.n_voxels} initial values")
    return v


def _gradient(s, yv, scenario, idx, dtype=None) -> np.ndarray:
    plan = get_plan(scenario, dtype)
    _subset_indices(idx, scenario)
    pred = forward_values(plan, np.asarray(s, dtype=np.complex128), idx)
    return adjoint_values(plan, pred - yv[idx], idx) / idx.size


# ------------------------------------------------------------------ public functions


def data_fidelity(s, y, scenario: ImagingScenario, subset=None, threads: int = 1, *, dtype=None) -> float:
    """(1/B) Σ ½|A_sub s − y_sub|² (solver.py:172-178)."""
    yv = _measurement_values(y, scenario)
    idx = _subset_or_all(subset, scenario)
    _subset_indices(idx, scenario)
    resid = forward_values(get_plan(scenario, dtype), _volume_values(s, scenario), idx) - yv[idx]
    return 0.5 * float(np.mean(np.abs(resid) ** 2))


def full_gradient(s, y, scenario: ImagingScenario, threads: int = 1, *, dtype=None) -> np.ndarray:
    """(1/M) A^H (A s − y) (solver.py:186-190)."""
    yv = _measurement_values(y, scenario)
    return _gradient(s, yv, scenario, np.arange(scenario.n_channels, dtype=np.int64), dtype)


def minibatch_gradient(s, y, scenario: ImagingScenario, subset, threads: int = 1, *, dtype=None) -> np.ndarray:
    """(1/B) A_sub^H (A_sub s − y_sub); the full subset is bitwise full_gradient (solver.py:193-203)."""
    if subset is None:
        raise ValueError("minibatch_gradient requires a non-empty channel subset")
    yv = _measurement_values(y, scenario)
    return _gradient(s, yv, scenario, _subset_or_all(subset, scenario), dtype)


def sample_minibatch(composition: MinibatchComposition, scenario: ImagingScenario, rng) -> ChannelSubset:
    """Structured Cartesian minibatch; same RNG call sequence as solver.py:206-225."""
    composition.validate_for(scenario)
    if not isinstance(rng, np.random.Generator):
        rng = np.random.default_rng(rng)
    T, R = scenario.array.n_tx, scenario.array.n_rx
    fs = np.sort(rng.choice(scenario.frequencies.count, composition.n_f, replace=False))
    ts = np.sort(rng.choice(T, composition.n_tx, replace=False))
    rs = np.sort(rng.choice(R, composition.n_rx, replace=False))
    return ChannelSubset((rs[None, None, :] + R * (ts[None, :, None] + T * fs[:, None, None])).reshape(-1))


def sample_flat(scenario: ImagingScenario, batch: int, rng) -> np.ndarray:
    """Flat uniform minibatch without replacement, ascending (BASELINE sampling)."""
    return np.sort(rng.choice(scenario.n_channels, batch, replace=False)).astype(np.int64)


def soft_threshold(v, alpha: float) -> np.ndarray:
    """v·max(|v|−α, 0)/|v|; magnitudes ≤ α map to exactly 0 (solver.py:228-241)."""
    if not (math.isfinite(alpha) and alpha >= 0):
        raise ValueError(f"alpha must be >= 0, got {alpha}")
    arr = np.asarray(v, dtype=np.complex128)
    dev = require_cuda(None)
    out = soft_threshold_dev(torch.from_numpy(np.ascontiguousarray(arr).ravel()).to(dev), alpha)
    return out.cpu().numpy().reshape(arr.shape)


def relative_magnitude_change(s_prev, s_next) -> float:
    """‖|s⁺| − |s|‖₂ / max(‖|s|‖₂, 1e-12) (solver.py:244-251)."""
    a = np.asarray(s_prev)
    b = np.asarray(s_next)
    if a.shape != b.shape:
        raise ValueError(f"iterate shapes differ: {a.shape} vs {b.shape}")
    dev = require_cuda(None)
    ta = torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128).ravel()).to(dev)
    tb = torch.from_numpy(np.ascontiguousarray(b, dtype=np.complex128).ravel()).to(dev)
    st = magnitude_change_dev(ta, tb).cpu().numpy()
    return float(math.sqrt(st[1])) / max(float(math.sqrt(st[0])), _ZERO_NORM_GUARD)


def check_termination(s_prev, s_next, tol: float) -> bool:
    return relative_magnitude_change(s_prev, s_next) < tol


# ------------------------------------------------------------------ device SPGM engine


class SPGMEngine:
    """GPU-resident SPGM state for one voxel slab.

    ``stage(idx)`` / ``sample_device(...)`` stage a batch and ``step_staged()`` enqueues one
    full iteration without synchronising. With a process group the forward partial sums
    over voxel slabs are all-reduced (one NCCL all-reduce of 2·B reals)
    before the adjoint.
    """

    def __init__(self, plan: DevicePlan, y: np.ndarray | torch.Tensor, eta: float, alpha: float,
                 initial: np.ndarray | torch.Tensor | None = None, process_group=None,
                 collective: str = "nccl"):
        if collective not in ("nccl", "peer", "auto"):
            raise ValueError("collective must be 'nccl', 'peer' or 'auto'")
        self.plan = plan
        self.eta = float(eta)
        self.alpha = float(alpha)
        self.pg = process_group
        # "peer": the forward's last reduce kernel all-reduces over NVLink itself (nf_forward_allreduce);
        # "nccl": nf_forward, then torch.distributed.all_reduce of the 2·B reals;
        # "auto": peer if its start-up check against NCCL passes on every rank, else NCCL
        self.collective = collective if process_group is not None else "nccl"
        if self.collective in ("peer", "auto"):
            from .sharding import connect_peer_allreduce, peer_allreduce_self_check

            # both steps run the same collectives on every rank and agree on their verdict over the group
            ok = connect_peer_allreduce(plan, process_group)
            ok = ok and peer_allreduce_self_check(plan, process_group)
            if not ok:
                if self.collective == "peer":
                    raise RuntimeError("peer all-reduce could not be connected or failed its start-up check")
                import warnings

                warnings.warn("peer all-reduce unavailable on this group; using NCCL")
                self.collective = "nccl"
            else:
                self.collective = "peer"
        dev = plan.device
        self.y = plan._as_dev(y, plan.M, "y")
        self.s = torch.zeros(plan.n_local, dtype=plan.torch_dtype, device=dev)
        if initial is not None:
            self.s.copy_(plan._as_dev(initial, plan.n_local, "initial"))
        self.s_next = torch.empty_like(self.s)
        self.ybuf = torch.empty(plan.max_batch, dtype=plan.torch_dtype, device=dev)
        self.stats = torch.zeros(4, dtype=torch.float64, device=dev)
        self.idx_dev = torch.empty(plan.max_batch, dtype=torch.int32, device=dev)
        # two persistent pinned staging buffers for host index lists (no per-call pinned allocation); a buffer is
        # reused only after the event recorded behind its last H2D copy has completed
        self._pinned = [None, None]
        self._pinned_ev = [None, None]
        self._pinned_next = 0
        # persistent loop (run_loop): records, state, index-table staging
        self._loop_rec = None
        self._loop_state = torch.zeros(4, dtype=torch.int32, device=dev)
        self._loop_pinned = None
        self._loop_tab = None
        self._loop_ev = None
        # chained persistent launches (run_loop_chained): per-slot records, state and index-table staging
        self._chain = [dict(rec=None, state=torch.zeros(4, dtype=torch.int32, device=dev), pinned=None, tab=None,
                            ev=None, h_state=torch.zeros(4, dtype=torch.int32).pin_memory(), h_rec=None, done=None)
                       for _ in range(2)]

    def _pinned_idx(self, n: int) -> tuple[torch.Tensor, int]:
        k = self._pinned_next
        self._pinned_next ^= 1
        if self._pinned_ev[k] is not None:
            self._pinned_ev[k].synchronize()
        if self._pinned[k] is None or self._pinned[k].numel() < n:
            self._pinned[k] = torch.empty(max(n, self.plan.max_batch), dtype=torch.int32).pin_memory()
        return self._pinned[k][:n], k

    def stage(self, idx) -> int:
        """Stage a host (numpy) or device index list; returns B."""
        if isinstance(idx, torch.Tensor) and idx.device == self.plan.device:
            t = idx.to(torch.int32)
        elif self.plan.try_structured(np.asarray(idx)):
            return self.plan.B
        else:
            arr = np.asarray(idx)
            B = int(arr.size)
            buf, k = self._pinned_idx(B)
            buf.numpy()[:] = arr.reshape(-1)  # int32 cast on the copy
            self.idx_dev[:B].copy_(buf, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.plan.device))
            self._pinned_ev[k] = ev
            t = self.idx_dev[:B]
        self.plan.prepare(t)
        return int(t.numel())

    def sample_device(self, seed: int, it: int | None, batch: int) -> None:
        """Device flat sampler; ``it=None`` uses the plan's device iteration counter."""
        self.plan.sample_flat(seed, it, batch, self.idx_dev)
        self.plan.prepare(self.idx_dev[:batch])

    def sample_device_structured(self, seed: int, it: int | None, composition) -> None:
        """Device structured sampler (a Cartesian n_f x n_tx x n_rx batch per iteration)."""
        c = composition
        self.plan.sample_structured(seed, it, c.n_f, c.n_tx, c.n_rx)

    def graph(self, seed: int, batch: int, pairs: int = 1, composition=None):
        """Capture ``2·pairs`` device-sampled SPGM iterations in one CUDA graph (an even count,
        so the iterate ends in the buffer it started in). Replays draw fresh batches from the
        plan's device iteration counter: flat batches of ``batch`` channels, or Cartesian
        ``composition`` batches. With a process group the NCCL all-reduce of the forward
        partials is captured into the graph as well."""

        def draw():
            if composition is None:
                self.sample_device(seed, None, batch)
            else:
                self.sample_device_structured(seed, None, composition)

        # one eager step outside capture so every kernel attribute is set (and NCCL is warm)
        draw()
        self.step_staged()
        torch.cuda.synchronize(self.plan.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(2 * pairs):
                draw()
                self.step_staged()
        return g

    def step_staged(self) -> None:
        """One iteration on the staged batch: forward, [allreduce], adjoint+prox, swap."""
        B = self.plan.B
        yb = self.ybuf[:B]
        if self.collective == "peer":
            self.plan.forward_allreduce(self.s, out=yb)
        else:
            self.plan.forward(self.s, out=yb)
            if self.pg is not None:
                torch.distributed.all_reduce(torch.view_as_real(yb), group=self.pg)
        self.plan.adjoint_prox(yb, self.y, self.s, self.s_next, self.eta / B, self.alpha, self.stats)
        self.s, self.s_next = self.s_next, self.s

    def run_loop(self, iters: int, table=None, seed: int = 0, iter0: int = 0, batch: int | None = None,
                 tol: float = 0.0, time_budget_s: float | None = None):
        """``iters`` SPGM iterations in one persistent launch (nf_spgm_loop): flat batches from ``table``
        ([iters, B] host array or device int32 tensor, subset order) or, with table=None, from the device
        sampler (``seed``, iteration numbers iter0, iter0 + 1, ...). Stops early on the tolerance test or
        the device-time budget. Returns (iterations run, reason 0/1/2, records [n, 6] float64 tensor on
        the device: the 4 statistics and the device time in ns since launch). Afterwards ``self.s`` is the
        latest iterate. Enqueued on the current stream; the caller synchronises (e.g. reading state)."""
        if self.pg is not None:
            raise RuntimeError("run_loop is single-GPU (voxel-slab ranks use step_staged with a collective)")
        dev = self.plan.device
        if table is not None:
            if not isinstance(table, torch.Tensor) or table.device != dev:
                arr = np.ascontiguousarray(np.asarray(table)[:iters], dtype=np.int32)
                buf = self._loop_table(arr.size)
                buf.numpy()[: arr.size] = arr.reshape(-1)
                tab = self._loop_dev_table(arr.size)
                tab[: arr.size].copy_(buf[: arr.size], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(torch.cuda.current_stream(dev))
                self._loop_ev = ev
                table = tab[: arr.size]
                batch = arr.shape[1]
            else:
                batch = int(table.shape[-1]) if table.dim() == 2 else int(batch)
                table = table.to(torch.int32).contiguous()
        if batch is None:
            raise ValueError("run_loop needs batch with the device sampler")
        if self._loop_rec is None or self._loop_rec.shape[0] < iters:
            self._loop_rec = torch.empty((max(iters, 64), 6), dtype=torch.float64, device=dev)
        self.plan.spgm_loop(table, iters, seed, iter0, batch, self.y, self.s, self.s_next, self.eta / batch,
                            self.alpha, tol, time_budget_s, self._loop_rec, self._loop_state)
        return self._loop_rec, self._loop_state

    def loop_result(self) -> tuple[int, int]:
        """(iterations run, reason) of the last run_loop (synchronises); swaps the iterate buffers so that
        ``self.s`` holds the latest iterate."""
        n, reason = (int(v) for v in self._loop_state[:2].cpu())
        if n % 2 == 1:
            self.s, self.s_next = self.s_next, self.s
        return n, reason

    def run_loop_chained(self, slot: int, prev_slot: int | None, iters: int, table=None, seed: int = 0,
                         iter0: int = 0, batch: int | None = None, tol: float = 0.0,
                         time_budget_s: float | None = None) -> None:
        """run_loop on slot ``slot``'s buffers through nf_spgm_loop_chained: if the launch on ``prev_slot``
        stopped early this one runs no iteration, and ``self.s`` holds the latest iterate after every launch, so
        the next launch can be enqueued before this one's state is read (chained_result)."""
        if self.pg is not None:
            raise RuntimeError("run_loop_chained is single-GPU")
        dev = self.plan.device
        c = self._chain[slot]
        if table is not None:
            arr = np.ascontiguousarray(np.asarray(table)[:iters], dtype=np.int32)
            if c["ev"] is not None:  # the slot's previous H2D copy has completed before its staging is rewritten
                c["ev"].synchronize()
            if c["pinned"] is None or c["pinned"].numel() < arr.size:
                c["pinned"] = torch.empty(max(arr.size, 4096), dtype=torch.int32).pin_memory()
            if c["tab"] is None or c["tab"].numel() < arr.size:
                c["tab"] = torch.empty(max(arr.size, 4096), dtype=torch.int32, device=dev)
            c["pinned"].numpy()[: arr.size] = arr.reshape(-1)
            c["tab"][: arr.size].copy_(c["pinned"][: arr.size], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(dev))
            c["ev"] = ev
            table = c["tab"][: arr.size]
            batch = arr.shape[1]
        if batch is None:
            raise ValueError("run_loop_chained needs batch with the device sampler")
        if c["rec"] is None or c["rec"].shape[0] < iters:
            c["rec"] = torch.empty((max(iters, 64), 6), dtype=torch.float64, device=dev)
        prev = None if prev_slot is None else self._chain[prev_slot]["state"]
        self.plan.spgm_loop(table, iters, seed, iter0, batch, self.y, self.s, self.s_next, self.eta / batch,
                            self.alpha, tol, time_budget_s, c["rec"], c["state"], prev_state=prev, chained=True)
        # state and records to pinned host memory right behind the launch, so reading them (chained_result) waits
        # for this launch only, not for the one enqueued after it
        if c["h_rec"] is None or c["h_rec"].shape[0] < iters:
            c["h_rec"] = torch.empty((max(iters, 64), 6), dtype=torch.float64).pin_memory()
        c["h_state"].copy_(c["state"], non_blocking=True)
        c["h_rec"][:iters].copy_(c["rec"][:iters], non_blocking=True)
        done = torch.cuda.Event()
        done.record(torch.cuda.current_stream(dev))
        c["done"] = done

    def chained_result(self, slot: int) -> tuple[int, int, np.ndarray]:
        """(iterations run, reason, records [n, 6] on the host) of the chained launch on ``slot``: waits for that
        launch (and its copies) only."""
        c = self._chain[slot]
        c["done"].synchronize()
        n, reason = (int(v) for v in c["h_state"][:2])
        return n, reason, c["h_rec"][:n].numpy()

    def _loop_table(self, n: int) -> torch.Tensor:
        if self._loop_ev is not None:
            self._loop_ev.synchronize()
        if self._loop_pinned is None or self._loop_pinned.numel() < n:
            self._loop_pinned = torch.empty(n, dtype=torch.int32).pin_memory()
        return self._loop_pinned

    def _loop_dev_table(self, n: int) -> torch.Tensor:
        if self._loop_tab is None or self._loop_tab.numel() < n:
            self._loop_tab = torch.empty(n, dtype=torch.int32, device=self.plan.device)
        return self._loop_tab

    def magnitude_change(self) -> float:
        if self.collective == "peer" and self.plan.comm_timed_out():
            raise RuntimeError("peer all-reduce: a rank stopped participating (flag wait timed out)")
        st = self.stats
        if self.pg is not None:
            st = st.clone()
            torch.distributed.all_reduce(st, group=self.pg)
        st = st.cpu().numpy()
        return float(math.sqrt(st[1])) / max(float(math.sqrt(st[0])), _ZERO_NORM_GUARD)

    def volume(self) -> np.ndarray:
        return self.s.to(torch.complex128).cpu().numpy()


def _solve(y, scenario: ImagingScenario, config: SolverConfig, initial, progress, stochastic: bool) -> SolveReport:
    yv = _measurement_values(y, scenario)
    m = scenario.n_channels
    s0 = None if initial is None else np.array(_volume_like(initial, scenario), dtype=np.complex128)
    dtype = config.dtype or default_dtype()
    plan = get_plan(scenario, dtype)
    eng = SPGMEngine(plan, yv, config.eta, config.alpha, initial=s0)
    rng = np.random.default_rng(config.rng_seed)
    full_idx = np.arange(m, dtype=np.int64)
    records: list[IterationRecord] = []
    termination = TERMINATION_MAX_ITERS
    iterations = 0
    staged_full = -1  # plan.stage_gen right after the full batch was staged

    def stage_iteration(k):  # host side of iteration k: draw (or reuse) its batch and stage it; returns B
        nonlocal staged_full
        if not stochastic:
            if staged_full != plan.stage_gen:
                eng.stage(full_idx)
                staged_full = plan.stage_gen
            return m
        if config.sampler == "device":
            if config.composition is not None:
                eng.sample_device_structured(config.rng_seed, k, config.composition)
                return config.composition.batch_size
            eng.sample_device(config.rng_seed, k, config.flat_batch)
            return config.flat_batch
        if config.sampler == "table":
            return eng.stage(np.asarray(config.index_table[k - 1]))
        if config.flat_batch is not None:
            return eng.stage(sample_flat(scenario, config.flat_batch, rng))
        return eng.stage(sample_minibatch(config.composition, scenario, rng).indices)

    t_start = time.perf_counter()
    loop_batch = _loop_batch(plan, config, scenario, stochastic) if progress is None and config.check_every == 1 \
        else None
    if loop_batch is not None:
        return _solve_persistent(eng, plan, config, scenario, stochastic, loop_batch, rng, t_start)
    if progress is None and config.check_every == 1:
        # Pipelined: iteration k+1 is drawn and launched before iteration k's statistics are read
        # (async D2H into a pinned double buffer), so host sampling and the read-back overlap the
        # GPU. If k terminates, the speculative step k+1 is dropped: its input, the iterate after
        # k, is still intact in the engine's other buffer, so results equal the serial loop's.
        stats_host = torch.empty((2, 4), dtype=torch.float64).pin_memory()
        events = [torch.cuda.Event(), torch.cuda.Event()]
        stream = torch.cuda.current_stream(plan.device)
        batch = {}
        t_launch = {}

        def launch(k):
            t_launch[k] = time.perf_counter()
            batch[k] = stage_iteration(k)
            eng.step_staged()
            stats_host[k % 2].copy_(eng.stats, non_blocking=True)
            events[k % 2].record(stream)

        launch(1)
        for k in range(1, config.max_iters + 1):
            if k < config.max_iters:
                launch(k + 1)
            events[k % 2].synchronize()
            st = stats_host[k % 2].tolist()
            change = math.sqrt(st[1]) / max(math.sqrt(st[0]), _ZERO_NORM_GUARD)
            iterations = k
            records.append(IterationRecord(k, change, time.perf_counter() - t_launch[k], batch[k]))
            stop = None
            if change < config.tol:
                stop = TERMINATION_TOLERANCE
            elif config.time_budget_s is not None and time.perf_counter() - t_start > config.time_budget_s:
                stop = TERMINATION_TIME_BUDGET
            if stop is not None:
                termination = stop
                if k < config.max_iters:  # drop the speculative step k+1
                    eng.s, eng.s_next = eng.s_next, eng.s
                break
        vol = eng.volume()
        return SolveReport(volume=ReflectivityVolume(vol, scenario.voxels), iterations=iterations,
                           wall_time_s=time.perf_counter() - t_start, per_iteration=records, termination=termination)

    for k in range(1, config.max_iters + 1):
        t_iter = time.perf_counter()
        if not stochastic:
            # the plan is shared (cached per scenario): a progress callback that evaluates the operator
            # on the same scenario re-stages it, so the full batch is staged again whenever that happened
            if staged_full != plan.stage_gen:
                eng.stage(full_idx)
                staged_full = plan.stage_gen
            B = m
        elif config.sampler == "device":
            if config.composition is not None:
                B = config.composition.batch_size
                eng.sample_device_structured(config.rng_seed, k, config.composition)
            else:
                B = config.flat_batch
                eng.sample_device(config.rng_seed, k, B)
        elif config.sampler == "table":
            B = eng.stage(np.asarray(config.index_table[k - 1]))
        elif config.flat_batch is not None:
            B = eng.stage(sample_flat(scenario, config.flat_batch, rng))
        else:
            B = eng.stage(sample_minibatch(config.composition, scenario, rng).indices)
        eng.step_staged()
        iterations = k
        check_now = (k % config.check_every == 0) or k == config.max_iters or progress is not None
        if check_now:
            change = eng.magnitude_change()
            records.append(IterationRecord(k, change, time.perf_counter() - t_iter, B))
        else:
            records.append(IterationRecord(k, float("nan"), time.perf_counter() - t_iter, B))
        if progress is not None:
            progress(k, eng.volume())
        if check_now and change < config.tol:
            termination = TERMINATION_TOLERANCE
            break
        if config.time_budget_s is not None and time.perf_counter() - t_start > config.time_budget_s:
            termination = TERMINATION_TIME_BUDGET
            break
    vol = eng.volume()
    wall = time.perf_counter() - t_start
    return SolveReport(
        volume=ReflectivityVolume(vol, scenario.voxels),
        iterations=iterations,
        wall_time_s=wall,
        per_iteration=records,
        termination=termination,
    )


LOOP_CHUNK = 256  # iterations per persistent launch (the host draws the next chunk's batches meanwhile)
LOOP_FIRST_CHUNK = 4
LOOP_MAX_ENTRIES = 1 << 28  # |B| x slab voxels per iteration up to which _solve uses the persistent loop


def _loop_batch(plan: DevicePlan, config: SolverConfig, scenario: ImagingScenario, stochastic: bool):
    """The batch size when this solve can run on the persistent device loop (nf_spgm_loop), else None.
    The loop computes flat batches; batches the per-iteration path would send to the separable kernels
    (Cartesian products with enough pairs, DevicePlan.try_structured) stay on that path, so every batch
    of a solve takes the same arithmetic either way."""
    import os

    if os.environ.get("NFGPU_LOOP", "1") == "0":
        return None
    from .plan import STRUCT_MIN_PAIRS, cartesian_factors

    def routes_flat(idx) -> bool:
        if plan.structured == "never":
            return True
        fac = cartesian_factors(idx, plan.n_tx, plan.n_rx)
        return fac is None or (plan.structured == "auto" and fac[1].size * fac[2].size < STRUCT_MIN_PAIRS)

    if not stochastic:
        B = scenario.n_channels
        ok = routes_flat(np.arange(B))
    elif config.sampler == "table":
        try:
            rows = np.asarray(config.index_table[: config.max_iters])
        except ValueError:  # ragged rows (batches of different sizes): the per-iteration path
            return None
        if rows.dtype == object or rows.ndim != 2:
            return None
        B = rows.shape[1]
        ok = all(routes_flat(r) for r in rows)
    elif config.composition is not None:
        c = config.composition
        B = c.batch_size
        ok = plan.structured == "never" or (plan.structured == "auto" and c.n_tx * c.n_rx < STRUCT_MIN_PAIRS)
    else:
        B = config.flat_batch
        ok = True
    # the loop pays off where launch latency is a visible share of an iteration; Large-sized iterations
    # (4096 x 1M entries, 4.7 ms) run as well pipelined from the host (e2e 4.72 vs 4.79 ms per iteration)
    if B * plan.n_local > LOOP_MAX_ENTRIES:
        return None
    return B if ok and plan.loop_eligible(B) else None


def _solve_persistent(eng: SPGMEngine, plan: DevicePlan, config: SolverConfig, scenario: ImagingScenario,
                      stochastic: bool, B: int, rng, t_start: float) -> SolveReport:
    """_solve on the persistent device loop: chunks of LOOP_CHUNK iterations per launch, each iteration's
    statistics, tolerance test (solver.py:302) and time-budget test on the device; the host draws the next
    chunk's batches with the reference's call sequence while the current chunk runs, and builds the
    IterationRecords (elapsed_seconds = device time of the iteration) from the records copied back once
    per chunk. Same iterates, records and termination as the per-iteration loop."""
    m = scenario.n_channels
    full = np.arange(m, dtype=np.int64)

    def draw(n):
        if not stochastic:
            return np.broadcast_to(full, (n, m))
        if config.sampler == "device":
            return None
        if config.sampler == "table":
            return None
        if config.flat_batch is not None:
            return np.stack([sample_flat(scenario, B, rng) for _ in range(n)])
        return np.stack([sample_minibatch(config.composition, scenario, rng).indices for _ in range(n)])

    records: list[IterationRecord] = []
    termination = TERMINATION_MAX_ITERS
    done = 0
    planned = 0  # iterations enqueued

    def enqueue(slot, prev_slot, n):
        nonlocal planned
        if config.sampler == "table":
            table = np.asarray(config.index_table[planned:planned + n])
        else:
            table = draw(n)
        budget = None
        if config.time_budget_s is not None:
            budget = max(0.0, config.time_budget_s - (time.perf_counter() - t_start))
        eng.run_loop_chained(slot, prev_slot, n, table=table, seed=config.rng_seed, iter0=planned + 1, batch=B,
                             tol=config.tol, time_budget_s=budget)
        planned += n

    # Chunks grow geometrically from LOOP_FIRST_CHUNK. Chunk j + 1 is drawn and enqueued before chunk j's state is
    # read (nf_spgm_loop_chained: it runs nothing if chunk j stopped early), so the host's sampling, record
    # building and launch overlap the GPU, which runs the chunks back to back.
    n = min(LOOP_FIRST_CHUNK, LOOP_CHUNK, config.max_iters)
    enqueue(0, None, n)
    slot = 0
    while True:
        n_next = min(2 * n, LOOP_CHUNK, config.max_iters - planned)
        if n_next > 0:
            enqueue(slot ^ 1, slot, n_next)
        k_run, reason, r = eng.chained_result(slot)
        t_prev = 0.0
        for i in range(k_run):
            st0, st1 = float(r[i, 0]), float(r[i, 1])
            change = math.sqrt(st1) / max(math.sqrt(st0), _ZERO_NORM_GUARD)
            records.append(IterationRecord(done + i + 1, change, (float(r[i, 4]) - t_prev) * 1e-9, B))
            t_prev = float(r[i, 4])
        done += k_run
        if reason == 1:
            termination = TERMINATION_TOLERANCE
            break
        if reason == 2 or (config.time_budget_s is not None and time.perf_counter() - t_start > config.time_budget_s):
            termination = TERMINATION_TIME_BUDGET
            break
        if n_next <= 0:
            break
        slot ^= 1
        n = n_next
    vol = eng.volume()
    return SolveReport(volume=ReflectivityVolume(vol, scenario.voxels), iterations=done,
                       wall_time_s=time.perf_counter() - t_start, per_iteration=records, termination=termination)


def pgm_solve(y, scenario: ImagingScenario, config: SolverConfig | None = None, initial=None,
              progress=None) -> SolveReport:
    """Full-batch proximal gradient from s⁰ = 0 (solver.py:332-346)."""
    config = config or SolverConfig()
    if config.composition is not None and not config.composition.is_full_for(scenario):
        raise ValueError("pgm_solve needs a full-batch config; use spgm_solve for minibatches")
    return _solve(y, scenario, config, initial, progress, stochastic=False)


def spgm_solve(y, scenario: ImagingScenario, config: SolverConfig | None = None, initial=None,
               progress=None) -> SolveReport:
    """Stochastic PGM, fresh minibatch per iteration (solver.py:349-365)."""
    config = config or SolverConfig()
    if config.composition is None and config.flat_batch is None and config.sampler != "table":
        raise ValueError("spgm_solve requires config.composition")
    if config.sampler == "table":
        for row in config.index_table[: config.max_iters]:
            _subset_indices(ChannelSubset(np.asarray(row)).indices, scenario)
    if config.composition is not None:
        config.composition.validate_for(scenario)
    if config.flat_batch is not None and config.flat_batch > scenario.n_channels:
        raise ValueError(f"flat_batch={config.flat_batch} exceeds M={scenario.n_channels}")
    return _solve(y, scenario, config, initial, progress, stochastic=True)


def lipschitz_estimate(scenario: ImagingScenario, n_iters: int = 50, rng_seed: int = 0, tol: float = 1e-9,
                       threads: int = 1, *, dtype=None) -> float:
    """λ_max((1/M) A^H A) by power iteration from the reference's start vector (solver.py:368-397)."""
    plan = get_plan(scenario, dtype)
    rng = np.random.default_rng(rng_seed)
    n, m = scenario.n_voxels, scenario.n_channels
    x0 = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    x0 /= np.linalg.norm(x0)
    x = plan._as_dev(x0, n, "x")
    plan.prepare_full()
    y = plan.vec(m)
    z = plan.vec(n)
    lam = 0.0
    for _ in range(n_iters):
        plan.forward(x, out=y)
        plan.adjoint(y, out=z, scale=1.0 / m)
        lam_new = float(torch.vdot(x, z).real)
        nz = float(torch.linalg.vector_norm(z))
        if nz == 0.0:
            return 0.0
        x = z / nz
        if lam > 0 and abs(lam_new - lam) <= tol * lam:
            lam = lam_new
            break
        lam = lam_new
    return lam
