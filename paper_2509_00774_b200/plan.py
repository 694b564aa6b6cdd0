"""Device-level wrapper around one ``nf_plan`` (include/nfgpu.h).

A :class:`DevicePlan` is the GPU replacement of the reference's cached
``_OperatorPlan`` (pkg/src/nfmimo/forward.py:183-211). It owns a frequency-free
per-(antenna, voxel) distance table for one voxel z-slab on one CUDA device.
Its methods take and return *device* torch tensors and enqueue work on the
current torch stream. Only the stream handle and raw pointers cross into the C ABI.
"""

from __future__ import annotations

import ctypes
import functools
import os

import numpy as np
import torch

from . import _lib
from .geometry import ImagingScenario

DTYPES = {"c64": (_lib.NF_C64, torch.complex64), "c128": (_lib.NF_C128, torch.complex128)}

# Structured (Cartesian) batches with at least this many (tx, rx) pairs per frequency take the
# separable kernels (nf_batch_prepare_structured); smaller ones stay on the flat path. On Large
# the two paths break even at 8 × 8 pairs (tools/time_structured.py, profiles/r01_structured.jsonl).
STRUCT_MIN_PAIRS = 64
STRUCT_POLICIES = ("auto", "always", "never")


def cartesian_factors(idx: np.ndarray, n_tx: int, n_rx: int):
    """(fs, ts, rs) when ``idx`` is exactly the sorted product Fs × Ts × Rs in (f, t, r) order,
    else None. That is the layout of the reference's sample_minibatch (solver.py:205-225) and
    of the full channel set (forward.py:233-236)."""
    idx = np.asarray(idx)
    if idx.ndim != 1 or idx.size == 0:
        return None
    idx = idx.astype(np.int64, copy=False)
    per_f = n_tx * n_rx
    fs = np.unique(idx // per_f)
    ts = np.unique((idx // n_rx) % n_tx)
    rs = np.unique(idx % n_rx)
    if fs.size * ts.size * rs.size != idx.size:
        return None
    expect = (rs[None, None, :] + n_rx * (ts[None, :, None] + n_tx * fs[:, None, None])).reshape(-1)
    if not np.array_equal(expect, idx):
        return None
    return fs.astype(np.int32), ts.astype(np.int32), rs.astype(np.int32)


def _dptr(x: np.ndarray):
    return x.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream(device: torch.device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def require_cuda(device=None) -> torch.device:
    """The GPU path is the only path: fail loudly without a CUDA device."""
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2509_00774_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback"
        )
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if dev.type != "cuda":
        raise RuntimeError(f"device must be a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


class DevicePlan:
    """One voxel slab [z_begin, z_end) of a scenario on one GPU."""

    def __init__(
        self,
        scenario: ImagingScenario,
        dtype: str = "c128",
        device=None,
        z_range: tuple[int, int] | None = None,
        max_batch: int | None = None,
        structured: str | None = None,
    ):
        """``structured``: "auto" (default; env NFGPU_STRUCTURED overrides) routes Cartesian
        host batches with >= STRUCT_MIN_PAIRS (tx, rx) pairs to the separable kernels,
        "always" routes every Cartesian host batch there, "never" keeps the flat path."""
        if dtype not in DTYPES:
            raise ValueError(f"dtype must be one of {sorted(DTYPES)}, got {dtype!r}")
        self.lib = _lib.load()
        self.device = require_cuda(device)
        self.scenario = scenario
        self.dtype_name = dtype
        self.nf_dtype, self.torch_dtype = DTYPES[dtype]
        self.real_dtype = torch.float32 if dtype == "c64" else torch.float64
        nx, ny, nz = scenario.voxels.dims
        z0, z1 = (0, nz) if z_range is None else (int(z_range[0]), int(z_range[1]))
        self.z_range = (z0, z1)
        self.n_local = nx * ny * (z1 - z0)
        self.vox_offset = nx * ny * z0
        self.structured = structured or os.environ.get("NFGPU_STRUCTURED", "auto")
        if self.structured not in STRUCT_POLICIES:
            raise ValueError(f"structured must be one of {STRUCT_POLICIES}, got {self.structured!r}")
        self.n_tx = scenario.array.n_tx
        self.n_rx = scenario.array.n_rx
        self.n_f = scenario.frequencies.count
        self.M = scenario.n_channels
        self.max_batch = self.M if max_batch is None else int(max_batch)

        tx = np.ascontiguousarray(scenario.array.tx_positions(), dtype=np.float64)
        rx = np.ascontiguousarray(scenario.array.rx_positions(), dtype=np.float64)
        freqs = np.ascontiguousarray(scenario.frequencies.values(), dtype=np.float64)
        pulse = scenario.pulse.evaluate(freqs).astype(np.complex128)
        pulse_ri = np.ascontiguousarray(np.stack([pulse.real, pulse.imag], axis=1).reshape(-1))
        corner = np.array(scenario.voxels.corner.as_array(), dtype=np.float64)
        spacing = np.array(scenario.voxels.spacing, dtype=np.float64)
        dims = (ctypes.c_int * 3)(nx, ny, nz)
        out = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            rc = self.lib.nf_plan_create(
                _dptr(tx), tx.shape[0], _dptr(rx), rx.shape[0], _dptr(freqs), _dptr(pulse_ri),
                freqs.size, float(scenario.c), _dptr(corner), _dptr(spacing), dims, z0, z1,
                self.nf_dtype, self.max_batch, ctypes.byref(out),
            )
        _lib.check(rc, "nf_plan_create")
        self._h = out
        self.B = 0
        self._idx = None  # keeps the staged index tensor alive
        self.staged_structured = False
        # bumped by every staging call: a caller that keeps a batch staged across calls it does not
        # control (the solver's full-batch PGM loop around a progress callback) re-stages on a change
        self.stage_gen = 0

    # ---------------------------------------------------------------- lifecycle
    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self.lib.nf_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    def info(self) -> dict:
        buf = (ctypes.c_int64 * 8)()
        _lib.check(self.lib.nf_plan_info(self._h, buf), "nf_plan_info")
        keys = ("n_local", "M", "tiles", "tx_group", "device_bytes", "fwd_window", "dtype", "launches")
        return dict(zip(keys, list(buf)))

    @property
    def launches(self) -> int:
        return self.info()["launches"]

    # ---------------------------------------------------------------- helpers
    def vec(self, n: int) -> torch.Tensor:
        return torch.empty(n, dtype=self.torch_dtype, device=self.device)

    def _as_dev(self, x, n: int, name: str) -> torch.Tensor:
        if isinstance(x, torch.Tensor):
            t = x.to(device=self.device, dtype=self.torch_dtype)
        else:
            t = torch.as_tensor(np.asarray(x), device=self.device).to(self.torch_dtype)
        t = t.contiguous()
        if t.shape != (n,):
            raise ValueError(f"{name}: expected shape ({n},), got {tuple(t.shape)}")
        return t

    # ---------------------------------------------------------------- operator
    def prepare(self, idx: torch.Tensor) -> None:
        """Stage channel subset ``idx`` (int32 device tensor, validated by the caller)."""
        if idx.dtype != torch.int32 or idx.device != self.device or not idx.is_contiguous():
            idx = idx.to(device=self.device, dtype=torch.int32).contiguous()
        B = int(idx.numel())
        _lib.check(self.lib.nf_batch_prepare(self._h, _ptr(idx), B, _stream(self.device)), "nf_batch_prepare")
        self.B = B
        self._idx = idx
        self.staged_structured = False
        self.stage_gen += 1

    def prepare_structured(self, fs, ts, rs) -> None:
        """Stage the Cartesian subset fs × ts × rs (sorted host index lists; the C ABI validates)."""
        arrs = [np.ascontiguousarray(np.asarray(a), dtype=np.int32) for a in (fs, ts, rs)]
        ip = [a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)) for a in arrs]
        _lib.check(
            self.lib.nf_batch_prepare_structured(self._h, ip[0], arrs[0].size, ip[1], arrs[1].size, ip[2],
                                                 arrs[2].size, _stream(self.device)),
            "nf_batch_prepare_structured",
        )
        self.B = int(arrs[0].size * arrs[1].size * arrs[2].size)
        self._idx = None
        self.staged_structured = True
        self.stage_gen += 1

    def prepare_full(self) -> None:
        """Stage all M channels (a Cartesian product; structured unless the policy is "never")."""
        if self.structured != "never":
            self.prepare_structured(np.arange(self.n_f), np.arange(self.n_tx), np.arange(self.n_rx))
        else:
            self.prepare(torch.arange(self.M, dtype=torch.int32, device=self.device))

    def try_structured(self, idx) -> bool:
        """Stage host index list ``idx`` through the separable path when it is a sorted Cartesian
        product and the policy allows; returns False (nothing staged) otherwise."""
        if self.structured == "never":
            return False
        fac = cartesian_factors(idx, self.n_tx, self.n_rx)
        if fac is None:
            return False
        if self.structured == "auto" and fac[1].size * fac[2].size < STRUCT_MIN_PAIRS:
            return False
        self.prepare_structured(*fac)
        return True

    def stage_host(self, idx) -> int:
        """Stage a host (numpy) index list in subset order; returns B."""
        idx = np.asarray(idx)
        if not self.try_structured(idx):
            self.prepare(torch.from_numpy(idx.astype(np.int32)).to(self.device))
        return self.B

    def forward(self, s: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """out[k] = Σ_{n in slab} A[m_k, n] s[n] (subset order)."""
        if out is None:
            out = self.vec(self.B)
        _lib.check(self.lib.nf_forward(self._h, _ptr(s), _ptr(out), _stream(self.device)), "nf_forward")
        return out

    # ---------------------------------------------------------------- peer all-reduce (multi-GPU)
    def comm_create(self, rank: int, world: int) -> bytes:
        """Allocate this rank's peer all-reduce slots; returns its CUDA IPC handle (64 bytes)."""
        h = ctypes.create_string_buffer(_lib.NF_IPC_HANDLE_BYTES)
        _lib.check(self.lib.nf_comm_create(self._h, int(rank), int(world), h), "nf_comm_create")
        return h.raw

    def comm_connect(self, handles: list[bytes]) -> None:
        """Map every rank's slots (``handles`` in rank order, from comm_create on each rank)."""
        if any(len(h) != _lib.NF_IPC_HANDLE_BYTES for h in handles):
            raise ValueError("comm_connect: every handle must be 64 bytes")
        buf = ctypes.create_string_buffer(b"".join(handles), len(handles) * _lib.NF_IPC_HANDLE_BYTES)
        _lib.check(self.lib.nf_comm_connect(self._h, buf), "nf_comm_connect")

    def forward_allreduce(self, s: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """forward() summed over every connected rank's slab by the fused peer all-reduce:
        out is the full A_B s on every rank (bitwise the same on all of them)."""
        if out is None:
            out = self.vec(self.B)
        _lib.check(self.lib.nf_forward_allreduce(self._h, _ptr(s), _ptr(out), _stream(self.device)),
                   "nf_forward_allreduce")
        return out

    def comm_timed_out(self) -> bool:
        """True if a peer flag wait gave up (synchronises with the device)."""
        v = ctypes.c_int(0)
        _lib.check(self.lib.nf_comm_status(self._h, ctypes.byref(v)), "nf_comm_status")
        return bool(v.value)

    def adjoint(self, r: torch.Tensor, out: torch.Tensor | None = None, ymeas: torch.Tensor | None = None,
                scale: float = 1.0) -> torch.Tensor:
        """out[n] = scale Σ_k conj(A[m_k, n]) (r[k] - ymeas[m_k])."""
        if out is None:
            out = self.vec(self.n_local)
        _lib.check(
            self.lib.nf_adjoint(self._h, _ptr(r), _ptr(ymeas), _ptr(out), float(scale), _stream(self.device)),
            "nf_adjoint",
        )
        return out

    def adjoint_prox(self, r, ymeas, s_in, s_out, eta_over_b: float, alpha: float, stats: torch.Tensor):
        _lib.check(
            self.lib.nf_adjoint_prox(
                self._h, _ptr(r), _ptr(ymeas), _ptr(s_in), _ptr(s_out), float(eta_over_b), float(alpha),
                _ptr(stats), _stream(self.device),
            ),
            "nf_adjoint_prox",
        )

    def sample_flat(self, seed: int, it: int | None, batch: int, out: torch.Tensor) -> torch.Tensor:
        """Flat batch for iteration ``it``; ``it=None`` uses (and advances) the plan's device
        iteration counter, so the call can be captured in a CUDA graph."""
        itv = _lib.NF_ITER_DEVICE if it is None else int(it)
        _lib.check(
            self.lib.nf_sample_flat(self._h, int(seed) & (2**64 - 1), itv, int(batch), _ptr(out),
                                    _stream(self.device)),
            "nf_sample_flat",
        )
        return out

    def sample_structured(self, seed: int, it: int | None, n_f: int, n_tx: int, n_rx: int,
                          lists: torch.Tensor | None = None) -> None:
        """Device structured sampler: draw and stage an n_f x n_tx x n_rx Cartesian batch
        (nf_sample_structured). ``it=None`` uses and advances the device iteration counter;
        ``lists`` (int32 device, n_f + n_tx + n_rx) receives the drawn [fs | ts | rs]."""
        itv = _lib.NF_ITER_DEVICE if it is None else int(it)
        _lib.check(
            self.lib.nf_sample_structured(self._h, int(seed) & (2**64 - 1), itv, int(n_f), int(n_tx), int(n_rx),
                                          _ptr(lists), _stream(self.device)),
            "nf_sample_structured",
        )
        self.B = int(n_f * n_tx * n_rx)
        self._idx = None
        self.staged_structured = True
        self.stage_gen += 1

    def spgm_loop(self, table: torch.Tensor | None, iters: int, seed: int, iter0: int, batch: int,
                  ymeas: torch.Tensor, s_a: torch.Tensor, s_b: torch.Tensor, eta_over_b: float, alpha: float,
                  tol: float, time_budget_s: float | None, records: torch.Tensor, state: torch.Tensor,
                  prev_state: torch.Tensor | None = None, chained: bool = False) -> None:
        """nf_spgm_loop: ``iters`` flat-batch SPGM iterations in one persistent launch (table: device int32
        [iters, batch] in subset order, or None for the device Feistel sampler). With ``prev_state`` (a tensor or
        None) and ``chained`` the launch goes through nf_spgm_loop_chained: it runs nothing when the previous launch stopped
        early, and it ends with the latest iterate in s_a."""
        args = (self._h, _ptr(table), int(iters), int(seed) & (2**64 - 1), int(iter0), int(batch), _ptr(ymeas),
                _ptr(s_a), _ptr(s_b), float(eta_over_b), float(alpha), float(tol),
                -1.0 if time_budget_s is None else float(time_budget_s), _ptr(records), _ptr(state))
        if chained:
            _lib.check(self.lib.nf_spgm_loop_chained(*args, _ptr(prev_state), _stream(self.device)),
                       "nf_spgm_loop_chained")
        else:
            _lib.check(self.lib.nf_spgm_loop(*args, _stream(self.device)), "nf_spgm_loop")
        self.B = int(batch)
        self._idx = None
        self.staged_structured = False
        self.stage_gen += 1

    def loop_eligible(self, batch: int) -> bool:
        """True when nf_spgm_loop can run this flat batch size (one forward window, <= 4096 channels)."""
        return 1 <= batch <= min(self.max_batch, 4096, self.fwd_chunk)

    @property
    def fwd_chunk(self) -> int:
        return int(self.info()["fwd_window"])

    def set_iter(self, it: int) -> None:
        _lib.check(self.lib.nf_plan_set_iter(self._h, int(it), _stream(self.device)), "nf_plan_set_iter")


def soft_threshold_dev(v: torch.Tensor, alpha: float, out: torch.Tensor | None = None) -> torch.Tensor:
    lib = _lib.load()
    nf = _lib.NF_C64 if v.dtype == torch.complex64 else _lib.NF_C128
    v = v.contiguous()
    out = torch.empty_like(v) if out is None else out
    _lib.check(lib.nf_soft_threshold(nf, _ptr(v), _ptr(out), v.numel(), float(alpha), _stream(v.device)),
               "nf_soft_threshold")
    return out


def magnitude_change_dev(a: torch.Tensor, b: torch.Tensor, stats: torch.Tensor | None = None) -> torch.Tensor:
    lib = _lib.load()
    nf = _lib.NF_C64 if a.dtype == torch.complex64 else _lib.NF_C128
    a, b = a.contiguous(), b.contiguous()
    if stats is None:
        stats = torch.empty(2, dtype=torch.float64, device=a.device)
    _lib.check(lib.nf_magnitude_change(nf, _ptr(a), _ptr(b), a.numel(), _ptr(stats), _stream(a.device)),
               "nf_magnitude_change")
    return stats


@functools.lru_cache(maxsize=4)
def cached_plan(scenario: ImagingScenario, dtype: str, device_index: int) -> DevicePlan:
    """Per-scenario plan cache, the analogue of the reference's lru_cache'd _plan (forward.py:190)."""
    return DevicePlan(scenario, dtype=dtype, device=torch.device("cuda", device_index))
