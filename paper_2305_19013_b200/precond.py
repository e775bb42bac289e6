"""Split block-Jacobi preconditioning M = L L^T (row F4; reference blockjacobi.py:1-183).

Setup (host, once per matrix): the dense diagonal blocks of A are factored
exactly (`chol`) or with zero fill-in (`ichol0`, with the reference's
diagonal-shift retries) -- the same numpy operations as the reference, so the
factors are bitwise the reference's.  The device keeps the dense factors L_b;
L^-1 / L^-T run as per-block substitutions (`ekcg_block_trsv`) and L / L^T
as a block-diagonal dense product (`ekcg_block_diag_apply`), over n x m
row-major blocks.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
from scipy.linalg import solve_triangular

from . import _lib
from .device import as_device, current_stream_ptr, get_device
from .linalg import Breakdown

__all__ = [
    "BlockJacobiFactor",
    "uniform_block_bounds",
    "build_block_jacobi",
    "forward_solve",
    "backward_solve",
    "apply_minv",
    "mult_l",
    "mult_lt",
    "aligned_with",
    "DevicePreconditioner",
]


@dataclass(frozen=True)
class BlockJacobiFactor:
    """Per-block lower-triangular factors over consecutive index ranges (blockjacobi.py:33-47)."""

    n: int
    block_bounds: tuple
    factors: tuple
    kind: str
    notes: tuple = field(default=())

    @property
    def nblocks(self):
        return len(self.block_bounds)


def uniform_block_bounds(n, nblocks):
    """Consecutive ranges; the first n mod nblocks get one extra row (blockjacobi.py:50-57)."""
    n, nblocks = int(n), int(nblocks)
    if nblocks < 1 or nblocks > n:
        raise ValueError(f"need 1 <= nblocks <= n, got {nblocks}, n={n}")
    base, extra = divmod(n, nblocks)
    edges = np.concatenate(([0], np.cumsum([base + 1] * extra + [base] * (nblocks - extra))))
    return tuple((int(edges[i]), int(edges[i + 1])) for i in range(nblocks))


def _diag_block(A, start, end):
    m = end - start
    out = np.zeros((m, m))
    for i in range(start, end):
        lo, hi = A.row_ptr[i], A.row_ptr[i + 1]
        cols = A.col_idx[lo:hi]
        inside = (cols >= start) & (cols < end)
        out[i - start, cols[inside] - start] = A.values[lo:hi][inside]
    return out


def _ichol0(block, pattern):
    """IC(0) on the lower pattern (blockjacobi.py:71-84)."""
    m = block.shape[0]
    L = np.where(pattern, np.tril(block), 0.0)
    for k in range(m):
        piv = L[k, k]
        if piv <= 0.0:
            raise Breakdown(f"nonpositive IC(0) pivot {piv:.3e} at local row {k}")
        L[k, k] = np.sqrt(piv)
        if k + 1 < m:
            col = np.where(pattern[k + 1:, k], L[k + 1:, k] / L[k, k], 0.0)
            L[k + 1:, k] = col
            L[k + 1:, k + 1:] -= np.where(pattern[k + 1:, k + 1:], np.outer(col, col), 0.0)
    return L


def build_block_jacobi(A, block_bounds, kind="chol", shift_retries=3):
    """Factor the diagonal blocks of A (blockjacobi.py:87-132)."""
    bounds = tuple((int(s), int(e)) for s, e in block_bounds)
    if bounds[0][0] != 0 or bounds[-1][1] != A.n:
        raise ValueError("block bounds must cover 0..n")
    for (s0, e0), (s1, _) in zip(bounds, bounds[1:]):
        if e0 != s1 or e0 <= s0:
            raise ValueError("block bounds must be consecutive, nonempty ranges")
    if bounds[-1][1] <= bounds[-1][0]:
        raise ValueError("block bounds must be consecutive, nonempty ranges")
    if kind not in ("chol", "ichol0"):
        raise ValueError(f"unknown factor kind {kind!r}")
    factors, notes = [], []
    for b, (start, end) in enumerate(bounds):
        block = _diag_block(A, start, end)
        if kind == "chol":
            try:
                factors.append(np.linalg.cholesky(block))
            except np.linalg.LinAlgError as exc:
                raise Breakdown(f"Cholesky failed on block {b + 1}: {exc}") from exc
            continue
        pattern = np.tril(block != 0.0)
        sigma = 1e-8 * float(np.max(np.diag(block)))
        shift = 0.0
        for attempt in range(shift_retries + 1):
            try:
                factors.append(_ichol0(block + shift * np.eye(block.shape[0]) if shift else block, pattern))
                if shift:
                    notes.append(f"block {b + 1}: IC(0) needed diagonal shift {shift:.3e}")
                break
            except Breakdown:
                if attempt == shift_retries:
                    raise Breakdown(f"IC(0) failed on block {b + 1} after {shift_retries} diagonal shifts")
                shift = sigma if shift == 0.0 else 2.0 * shift
    return BlockJacobiFactor(A.n, bounds, tuple(factors), kind, tuple(notes))


def aligned_with(F, partition):
    """Every preconditioner block inside one subdomain (blockjacobi.py:176-183)."""
    owner = partition.owner()
    return all(np.all(owner[s:e] == owner[s]) for s, e in F.block_bounds)


class DevicePreconditioner:
    """Device copy of a block-Jacobi factor (ours or the reference's, duck-typed):
    L_b and L_b^-1 per block, applied by the block-diagonal product kernel."""

    FORWARD, BACKWARD, MULT_L, MULT_LT = range(4)

    def __init__(self, F, device=None):
        self.device = get_device(device)
        self.n = int(F.n)
        bounds = tuple(F.block_bounds)
        starts = np.array([s for s, _ in bounds] + [bounds[-1][1]], dtype=np.int32)
        sizes = np.diff(starts).astype(np.int64)
        offs = np.concatenate(([0], np.cumsum(sizes * sizes)))[:-1].astype(np.int64)
        Ls = [np.ascontiguousarray(np.asarray(L, dtype=np.float64)) for L in F.factors]
        row_block = np.repeat(np.arange(len(bounds), dtype=np.int32), sizes)
        to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(self.device)
        self.L = to(np.concatenate([L.reshape(-1) for L in Ls]))
        self.offs, self.starts, self.row_block = to(offs), to(starts), to(row_block)
        self.bounds = bounds
        self.host = F

    def apply(self, mode, X, ldx, Y, ldy, m, live=None, stream=None):
        """Y = op(X) for op in {L^-1, L^-T, L, L^T} on an n x m block.

        The solves run by substitution (ekcg_block_trsv, like solve_triangular);
        the products by the block-diagonal dense kernel (Y must differ from X)."""
        transpose = 1 if mode in (self.BACKWARD, self.MULT_LT) else 0
        st = current_stream_ptr(self.device) if stream is None else stream
        xp = X if isinstance(X, int) else X.data_ptr()
        yp = Y if isinstance(Y, int) else Y.data_ptr()
        if mode in (self.FORWARD, self.BACKWARD):
            _lib.call("ekcg_block_trsv", self.L.data_ptr(), self.offs.data_ptr(), self.starts.data_ptr(),
                      len(self.bounds), transpose, xp, ldx, yp, ldy, m, live, st)
        else:
            _lib.call("ekcg_block_diag_apply", self.L.data_ptr(), self.offs.data_ptr(), self.starts.data_ptr(),
                      self.row_block.data_ptr(), transpose, xp, ldx, yp, ldy, self.n, m, live, st)


def _device_pc(F):
    if isinstance(F, DevicePreconditioner):
        return F
    return DevicePreconditioner(F)


def _apply_api(F, v, modes):
    pc = _device_pc(F)
    vt, back = as_device(v)
    if vt.shape[0] != pc.n:
        raise ValueError(f"expected leading dimension {pc.n}, got {tuple(vt.shape)}")
    X = vt.reshape(pc.n, -1).contiguous()
    m = X.shape[1]
    for mode in modes:
        Y = torch.empty_like(X)
        pc.apply(mode, X, m, Y, m, m)
        X = Y
    return back(X.reshape(vt.shape))


def forward_solve(F, v):
    """L^-1 v block by block (blockjacobi.py:145-147), on the device."""
    return _apply_api(F, v, [DevicePreconditioner.FORWARD])


def backward_solve(F, v):
    """L^-T v block by block (blockjacobi.py:150-152), on the device."""
    return _apply_api(F, v, [DevicePreconditioner.BACKWARD])


def apply_minv(F, v):
    """M^-1 v = L^-T L^-1 v (blockjacobi.py:155-157), on the device."""
    return _apply_api(F, v, [DevicePreconditioner.FORWARD, DevicePreconditioner.BACKWARD])


def mult_l(F, v):
    return _apply_api(F, v, [DevicePreconditioner.MULT_L])


def mult_lt(F, v):
    return _apply_api(F, v, [DevicePreconditioner.MULT_LT])
