"""Numpy restatement of the reference's operator and solver (TEST INFRASTRUCTURE ONLY).

Two evaluators of the same operator:

* ``TableOperator`` — the reference's own CPU algorithm (forward.py:183-336):
  per-scenario complex128 phasor tables u[f,t,n], v[f,r,n] split so that
  A[m,n] = p_f·u[f,t,n]·v[f,r,n]; forward = per-(f,t) group elementwise product
  then one length-N dot per receiver; adjoint = per-frequency partials (GEMM for
  rectangular groups, gather+matvec otherwise) summed in ascending frequency.
  This is the CPU baseline of bench.py (kind "port").
* ``direct_forward`` / ``direct_adjoint`` — chunked evaluation of the propagation
  formula (forward.py:142-155) without tables, for sizes whose tables do not fit
  in host memory (Large: 206 GB). Used for spot checks.

Plus the solver pieces: soft threshold (solver.py:228-241), relative magnitude
change (solver.py:244-251), the SPGM loop (solver.py:259-318) driven by an
explicit index sequence, and the power-iteration Lipschitz estimate
(solver.py:368-397).

Inputs are plain arrays (``Geom``), so the oracle shares no code with the product.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Geom:
    tx: np.ndarray      # (T, 3) float64
    rx: np.ndarray      # (R, 3) float64
    freqs: np.ndarray   # (F,)  float64, np.linspace
    pulse: np.ndarray   # (F,)  complex128
    centers: np.ndarray  # (N, 3) float64, x fastest
    c: float

    @property
    def T(self):
        return self.tx.shape[0]

    @property
    def R(self):
        return self.rx.shape[0]

    @property
    def F(self):
        return self.freqs.size

    @property
    def M(self):
        return self.F * self.T * self.R

    @property
    def N(self):
        return self.centers.shape[0]


def centers_of(corner, spacing, dims, z_range=None) -> np.ndarray:
    """Voxel centres corner + i·spacing, x fastest (geometry.py:194-207)."""
    nx, ny, nz = dims
    z0, z1 = (0, nz) if z_range is None else z_range
    n = np.arange(nx * ny * (z1 - z0))
    out = np.empty((n.size, 3))
    out[:, 0] = corner[0] + (n % nx) * spacing[0]
    out[:, 1] = corner[1] + ((n // nx) % ny) * spacing[1]
    out[:, 2] = corner[2] + (z0 + n // (nx * ny)) * spacing[2]
    return out


def geom_from_scenario(scn, z_range=None) -> Geom:
    """Duck-typed: accepts a reference nfmimo.ImagingScenario or the product's."""
    v = scn.voxels
    freqs = scn.frequencies.values()
    return Geom(
        tx=np.asarray(scn.array.tx_positions(), dtype=np.float64).reshape(-1, 3),
        rx=np.asarray(scn.array.rx_positions(), dtype=np.float64).reshape(-1, 3),
        freqs=np.asarray(freqs, dtype=np.float64),
        pulse=np.asarray(scn.pulse.evaluate(freqs), dtype=np.complex128),
        centers=centers_of(v.corner.as_array(), v.spacing, v.dims, z_range),
        c=float(scn.c),
    )


def decode(m, T, R):
    """m → (fi, ti, ri), receiver fastest (geometry.py:316-324)."""
    m = np.asarray(m, dtype=np.int64)
    return m // (T * R), (m // R) % T, m % R


# ---------------------------------------------------------------- direct formula


def element_row(g: Geom, m: int, centers: np.ndarray | None = None) -> np.ndarray:
    """A[m, :] from distances (forward.py:142-155)."""
    centers = g.centers if centers is None else centers
    fi, ti, ri = (int(v) for v in decode(m, g.T, g.R))
    f = g.freqs[fi]
    dt = np.sqrt(np.sum((centers - g.tx[ti]) ** 2, axis=1))
    dr = np.sqrt(np.sum((centers - g.rx[ri]) ** 2, axis=1))
    return g.pulse[fi] * np.exp(-1j * (2.0 * math.pi / g.c) * f * (dt + dr)) / (4.0 * math.pi * dt * dr)


def _dist(centers, pos):
    return np.sqrt(np.sum((centers[:, None, :] - pos[None, :, :]) ** 2, axis=2))  # (n, k)


def direct_forward(g: Geom, s: np.ndarray, idx, chunk: int = 8192) -> np.ndarray:
    """y[k] = Σ_n A[m_k, n] s_n by the formula, chunked over voxels (no tables)."""
    fi, ti, ri = decode(idx, g.T, g.R)
    w = (2.0 * math.pi / g.c) * g.freqs[fi]
    y = np.zeros(len(fi), dtype=np.complex128)
    for a in range(0, g.N, chunk):
        cen = g.centers[a:a + chunk]
        dt = _dist(cen, g.tx)  # (n, T)
        dr = _dist(cen, g.rx)
        d_sum = dt[:, ti] + dr[:, ri]  # (n, B)
        A = np.exp(-1j * w[None, :] * d_sum) / (4.0 * math.pi * dt[:, ti] * dr[:, ri])
        y += s[a:a + chunk] @ A
    return g.pulse[fi] * y


def direct_adjoint(g: Geom, r: np.ndarray, idx, voxels=None, chunk: int = 4096) -> np.ndarray:
    """x[n] = Σ_k conj(A[m_k, n]) r_k by the formula, for all voxels or a given subset."""
    fi, ti, ri = decode(idx, g.T, g.R)
    w = (2.0 * math.pi / g.c) * g.freqs[fi]
    coef = np.conj(g.pulse[fi]) * np.asarray(r, dtype=np.complex128)
    cen_all = g.centers if voxels is None else g.centers[np.asarray(voxels)]
    out = np.empty(cen_all.shape[0], dtype=np.complex128)
    for a in range(0, cen_all.shape[0], chunk):
        cen = cen_all[a:a + chunk]
        dt = _dist(cen, g.tx)
        dr = _dist(cen, g.rx)
        d_sum = dt[:, ti] + dr[:, ri]
        A_conj = np.exp(1j * w[None, :] * d_sum) / (4.0 * math.pi * dt[:, ti] * dr[:, ri])
        out[a:a + chunk] = A_conj @ coef
    return out


# ---------------------------------------------------------------- the reference's table algorithm


class TableOperator:
    """Phasor-table operator exactly as the reference computes it (forward.py:183-336)."""

    def __init__(self, g: Geom):
        self.g = g
        w = 2.0 * math.pi * g.freqs / g.c

        def build(pos):
            tab = np.empty((g.F, pos.shape[0], g.N), dtype=np.complex128)
            for a in range(pos.shape[0]):
                d = np.sqrt(np.sum((g.centers - pos[a]) ** 2, axis=1))
                amp = 1.0 / (2.0 * math.sqrt(math.pi) * d)
                for f in range(g.F):
                    tab[f, a] = np.exp(-1j * w[f] * d) * amp
            return tab

        self.pulse = g.pulse
        self.tx_tab = build(g.tx)
        self.rx_tab = build(g.rx)

    @staticmethod
    def table_bytes(g: Geom) -> int:
        return 16 * g.F * (g.T + g.R) * g.N

    def _groups(self, idx):
        """Runs of equal (f, t) in (f, t, r) order, keeping output positions (forward.py:240-258)."""
        fi, ti, ri = decode(idx, self.g.T, self.g.R)
        order = np.lexsort((ri, ti, fi))
        key = (fi * self.g.T + ti)[order]
        cuts = np.flatnonzero(np.diff(key)) + 1
        out = []
        for pos in np.split(order, cuts):
            out.append((int(fi[pos[0]]), int(ti[pos[0]]), ri[pos], pos))
        return out

    @staticmethod
    def _run(tasks, threads):
        if threads > 1 and len(tasks) > 1:
            with ThreadPoolExecutor(max_workers=min(threads, len(tasks))) as ex:
                return list(ex.map(lambda t: t(), tasks))
        return [t() for t in tasks]

    def forward(self, s: np.ndarray, idx, threads: int = 1) -> np.ndarray:
        idx = np.asarray(idx, dtype=np.int64)
        out = np.empty(idx.size, dtype=np.complex128)

        def task_for(f, t, rs, pos):
            def run():
                wrow = self.tx_tab[f, t] * s
                rows = self.rx_tab[f]
                p = self.pulse[f]
                for r, k in zip(rs, pos):
                    out[k] = p * np.dot(wrow, rows[r])
            return run

        self._run([task_for(*grp) for grp in self._groups(idx)], threads)
        return out

    def adjoint(self, r: np.ndarray, idx, threads: int = 1) -> np.ndarray:
        idx = np.asarray(idx, dtype=np.int64)
        r = np.asarray(r, dtype=np.complex128)
        g = self.g
        by_f: dict[int, list] = {}
        for grp in self._groups(idx):
            by_f.setdefault(grp[0], []).append(grp)

        def task_for(f, grps):
            def run():
                ts = np.array([q[1] for q in grps])
                p = self.pulse[f]
                trows = self.tx_tab[f] if ts.size == g.T else self.tx_tab[f][ts]
                rs0 = grps[0][2]
                if all(np.array_equal(q[2], rs0) for q in grps):
                    rrows = self.rx_tab[f] if rs0.size == g.R else self.rx_tab[f][rs0]
                    coef = np.conj(np.array([r[q[3]] for q in grps]) * np.conj(p))
                    return np.conj(np.einsum("tn,tn->n", trows, coef @ rrows))
                acc = np.zeros(g.N, dtype=np.complex128)
                for q, trow in zip(grps, trows):
                    acc += trow * (np.conj(r[q[3]] * np.conj(p)) @ self.rx_tab[f][q[2]])
                return np.conj(acc)
            return run

        fs = sorted(by_f)
        parts = self._run([task_for(f, by_f[f]) for f in fs], threads)
        out = np.zeros(g.N, dtype=np.complex128)
        for part in parts:
            out += part
        return out


# ---------------------------------------------------------------- solver pieces


def soft_threshold(v, alpha: float) -> np.ndarray:
    if not (math.isfinite(alpha) and alpha >= 0):
        raise ValueError(f"alpha must be >= 0, got {alpha}")
    v = np.asarray(v, dtype=np.complex128)
    mag = np.abs(v)
    scale = np.zeros(v.shape)
    keep = mag > alpha
    scale[keep] = (mag[keep] - alpha) / mag[keep]
    return v * scale


def relative_magnitude_change(a, b) -> float:
    a, b = np.abs(np.asarray(a)), np.abs(np.asarray(b))
    return float(np.linalg.norm(b - a)) / max(float(np.linalg.norm(a)), 1e-12)


def spgm(op, y: np.ndarray, eta: float, alpha: float, index_seq, s0=None, threads: int = 1,
         record=None):
    """s ← soft(s − η·A_B^H(A_B s − y_B)/B, α) for each index set (solver.py:259-318, tol disabled)."""
    s = np.zeros(op.g.N, dtype=np.complex128) if s0 is None else np.array(s0, dtype=np.complex128)
    changes = []
    for idx in index_seq:
        idx = np.asarray(idx, dtype=np.int64)
        resid = op.forward(s, idx, threads) - y[idx]
        grad = op.adjoint(resid, idx, threads) / idx.size
        s_next = soft_threshold(s - eta * grad, alpha)
        changes.append(relative_magnitude_change(s, s_next))
        if record is not None:
            record(s_next)
        s = s_next
    return s, changes


def lipschitz(op, n_iters: int = 50, rng_seed: int = 0, tol: float = 1e-9, threads: int = 1) -> float:
    g = op.g
    rng = np.random.default_rng(rng_seed)
    x = rng.standard_normal(g.N) + 1j * rng.standard_normal(g.N)
    x /= np.linalg.norm(x)
    full = np.arange(g.M)
    lam = 0.0
    for _ in range(n_iters):
        z = op.adjoint(op.forward(x, full, threads), full, threads) / g.M
        lam_new = float(np.real(np.vdot(x, z)))
        nz = np.linalg.norm(z)
        if nz == 0.0:
            return 0.0
        x = z / nz
        if lam > 0 and abs(lam_new - lam) <= tol * lam:
            return lam_new
        lam = lam_new
    return lam


def flat_index_sequence(M: int, B: int, iters: int, seed: int) -> list:
    """np.sort(rng.choice(M, B, replace=False)) per iteration from one persistent generator."""
    rng = np.random.default_rng(seed)
    return [np.sort(rng.choice(M, B, replace=False)) for _ in range(iters)]


def host_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
