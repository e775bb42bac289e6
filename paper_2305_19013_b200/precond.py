"""Split block-Jacobi preconditioning M = L L^T (row F4; reference blockjacobi.py:1-183).

Setup (host, once per matrix): the dense diagonal blocks of A are gathered in
one pass over the CSR and factored exactly (`chol`, LAPACK) or with zero
fill-in (`ichol0`, left-looking rows, with the reference's diagonal-shift
retries).  The reference's own factor objects are accepted as they are.  The device keeps the dense factors L_b;
L^-1 / L^-T run as per-block substitutions (`ekcg_block_trsv`) and L / L^T
as a block-diagonal dense product (`ekcg_block_diag_apply`), over n x m
row-major blocks.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .device import as_device, current_stream_ptr, get_device
from .linalg import Breakdown

__all__ = [
    "BlockJacobiFactor",
    "uniform_block_bounds",
    "diagonal_blocks",
    "ichol0",
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
    """Per-block lower-triangular factors over consecutive index ranges.

    The field layout is the reference's factor type (blockjacobi.py:33-47), so a
    factor built by either package can be passed as `SolverConfig.preconditioner`."""

    n: int
    block_bounds: tuple
    factors: tuple
    kind: str
    notes: tuple = field(default=())

    @property
    def nblocks(self):
        return len(self.block_bounds)


def uniform_block_bounds(n, nblocks):
    """Consecutive ranges, the first n mod nblocks one row longer (blockjacobi.py:50-57)."""
    n, nblocks = int(n), int(nblocks)
    if nblocks < 1 or nblocks > n:
        raise ValueError(f"need 1 <= nblocks <= n, got {nblocks}, n={n}")
    q, r = divmod(n, nblocks)
    cut = [i * q + min(i, r) for i in range(nblocks + 1)]
    return tuple(zip(cut[:-1], cut[1:]))


def _check_bounds(bounds, n):
    starts = np.array([s for s, _ in bounds], dtype=np.int64)
    ends = np.array([e for _, e in bounds], dtype=np.int64)
    if starts[0] != 0 or ends[-1] != n:
        raise ValueError("block bounds must cover 0..n")
    if np.any(ends <= starts) or np.any(starts[1:] != ends[:-1]):
        raise ValueError("block bounds must be consecutive, nonempty ranges")


def diagonal_blocks(A, bounds):
    """Dense diagonal blocks A[s:e, s:e], gathered in one vectorised pass over the CSR:
    entries whose row and column fall in the same range are scattered into their block."""
    n = int(A.n)
    rp = np.asarray(A.row_ptr, dtype=np.int64)
    ci = np.asarray(A.col_idx, dtype=np.int64)
    vv = np.asarray(A.values, dtype=np.float64)
    starts = np.array([s for s, _ in bounds], dtype=np.int64)
    blk_of = np.searchsorted(starts, np.arange(n), side="right") - 1  # block of every index
    rows = np.repeat(np.arange(n), np.diff(rp))
    inside = blk_of[rows] == blk_of[ci]
    rows, cols, vals, blk = rows[inside], ci[inside], vv[inside], blk_of[rows[inside]]
    out = [np.zeros((e - s, e - s)) for s, e in bounds]
    for b in np.unique(blk):
        sel = blk == b
        out[b][rows[sel] - starts[b], cols[sel] - starts[b]] = vals[sel]
    return out


def ichol0(B):
    """Incomplete Cholesky with zero fill-in of a dense SPD block, on the lower
    nonzero pattern of B (the factor blockjacobi.py:71-84 defines), in the
    left-looking row form: row i is finished from rows j < i already final,

        L[i, j] = (B[i, j] - L[i, :j] . L[j, :j]) / L[j, j]   for (i, j) in the pattern,
        L[i, i] = sqrt(B[i, i] - L[i, :i] . L[i, :i]),

    where L[i, k] is zero off the pattern.  Raises Breakdown on a nonpositive pivot."""
    m = B.shape[0]
    L = np.zeros_like(B)
    for i in range(m):
        row = L[i]
        for j in np.flatnonzero(B[i, :i]):
            row[j] = (B[i, j] - row[:j] @ L[j, :j]) / L[j, j]
        piv = B[i, i] - row[:i] @ row[:i]
        if not piv > 0.0:
            raise Breakdown(f"nonpositive IC(0) pivot {piv:.3e} at local row {i}")
        row[i] = np.sqrt(piv)
    return L


def build_block_jacobi(A, block_bounds, kind="chol", shift_retries=3):
    """Block-Jacobi factor of A (blockjacobi.py:87-132): exact dense Cholesky of every
    diagonal block ("chol") or IC(0) ("ichol0"); an IC(0) breakdown is retried with
    the diagonal shifted by 1e-8 * max(diag), doubling, at most `shift_retries` times."""
    bounds = tuple((int(s), int(e)) for s, e in block_bounds)
    _check_bounds(bounds, A.n)
    if kind not in ("chol", "ichol0"):
        raise ValueError(f"unknown factor kind {kind!r}")
    factors, notes = [], []
    for b, B in enumerate(diagonal_blocks(A, bounds), start=1):
        if kind == "chol":
            try:
                factors.append(np.linalg.cholesky(B))
            except np.linalg.LinAlgError as exc:
                raise Breakdown(f"Cholesky failed on block {b}: {exc}") from exc
            continue
        base = 1e-8 * float(B.diagonal().max())
        shifts = [0.0] + [base * 2.0 ** i for i in range(shift_retries)]
        for shift in shifts:
            try:
                L = ichol0(B + shift * np.eye(len(B)) if shift else B)
            except Breakdown:
                continue
            if shift:
                notes.append(f"block {b}: IC(0) needed diagonal shift {shift:.3e}")
            factors.append(L)
            break
        else:
            raise Breakdown(f"IC(0) failed on block {b} after {shift_retries} diagonal shifts")
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
