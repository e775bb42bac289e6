"""CPU oracle for the enlarged-CG hot loop -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference `ekcg` package's solver
path (SRE-CG / SRE-CG2 / truncated / restarted / flexible, MSDO variants) plus
this project's s-step extension.  It exists to check the CUDA product path:
only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline legs may
import it.  The product package never imports it and has no CPU fallback.

Parity pin: `tests/test_oracle_golden.py` checks every function here against
golden vectors produced by running the real reference (imported from
/root/reference in the build container) -- see `tests/golden/make_golden.py`.
Where the reference uses numpy/BLAS primitives the restatement uses the same
primitive in the same order, so results are bitwise identical to the
reference on the same host (the golden tests assert that).  The s-step
variant (s > 1) has no reference counterpart: it is "parity unpinned" beyond
its s = 1 reduction, which is bitwise SRE-CG2.

Citations are `file:line` into the reference tree `pkg/src/ekcg/`.
"""

from __future__ import annotations

import numpy as np
from scipy.linalg import solve_triangular

# linalg.py:25 -- spmm processes at most this many columns per gather pass.
COLUMN_SLAB = 64


class OracleBreakdown(Exception):
    """Mirror of `Breakdown` (linalg.py:28-34)."""


# ---------------------------------------------------------------------------
# Sparse products (linalg.py:133-152).  The association produced by
# np.add.reduceat is y_i = p_0 + pairwise(p_1 .. p_k) with p_j = v_j * x_cj
# rounded separately (no FMA); the CUDA kernels reproduce it bit for bit.
# ---------------------------------------------------------------------------

def csr_spmv(row_ptr, col_idx, values, x):
    """y = A x, same primitive as linalg.py:133-138."""
    prod = values * x[col_idx]
    return np.add.reduceat(prod, row_ptr[:-1])


def csr_spmm(row_ptr, col_idx, values, X):
    """Y = A X column-slab by column-slab, as linalg.py:141-152."""
    n, m = X.shape
    Y = np.empty((n, m))
    starts = row_ptr[:-1]
    scale = values[:, None]
    for c0 in range(0, m, COLUMN_SLAB):
        c1 = min(m, c0 + COLUMN_SLAB)
        Y[:, c0:c1] = np.add.reduceat(scale * X[col_idx, c0:c1], starts, axis=0)
    return Y


def pairwise_tail(vals):
    """numpy's pairwise summation (loops_utils.h) of a 1-D float sequence.

    Used only by the bit-exactness tests to spell out the association
    `p_0 + pairwise_tail(p_1..p_k)` that csr_spmv/csr_spmm realise.
    """
    n = len(vals)
    if n < 8:
        acc = -0.0
        for v in vals:
            acc = acc + v
        return acc
    if n <= 128:
        r = list(vals[:8])
        i = 8
        stop = n - (n % 8)
        while i < stop:
            for j in range(8):
                r[j] = r[j] + vals[i + j]
            i += 8
        acc = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            acc = acc + vals[i]
            i += 1
        return acc
    half = n // 2
    half -= half % 8
    return pairwise_tail(vals[:half]) + pairwise_tail(vals[half:])


# ---------------------------------------------------------------------------
# T^t split and halving (partition.py:44-65)
# ---------------------------------------------------------------------------

def split_block(owner, t, v):
    """n x t block with v copied into column owner[i] of row i (partition.py:48-55)."""
    n = owner.shape[0]
    out = np.zeros((n, t))
    out[np.arange(n), owner] = v
    return out


def halve_owner(owner):
    """Subdomains (2i, 2i+1) merge into i (partition.py:57-65)."""
    return owner // 2


# ---------------------------------------------------------------------------
# Small dense kernels (linalg.py:164-201, aortho.py:21-22,74-79)
# ---------------------------------------------------------------------------

def small_cholesky(B, breakdown_tol=1e-14):
    """Upper R with R^T R = B, row-oriented (linalg.py:164-184)."""
    m = B.shape[0]
    scale = float(np.max(np.abs(np.diag(B)))) if m else 0.0
    R = np.zeros((m, m))
    for j in range(m):
        col = R[:j, j]
        piv = B[j, j] - col @ col
        if not np.isfinite(piv) or piv <= breakdown_tol * scale:
            raise OracleBreakdown(f"pivot {piv:.3e} at column {j} (scale {scale:.3e})")
        R[j, j] = np.sqrt(piv)
        if j + 1 < m:
            R[j, j + 1:] = (B[j, j + 1:] - col @ R[:j, j + 1:]) / R[j, j]
    return R


def right_tri_solve(X, R):
    """Y with Y R = X for upper R (linalg.py:187-196)."""
    if np.any(np.diag(R) == 0.0):
        raise np.linalg.LinAlgError("singular triangular factor")
    return solve_triangular(R, X.T, trans="T", lower=False).T


def symmetrize(G):
    return 0.5 * (G + G.T)


def unit_columns(W):
    """Column scaling entering Pre-CholQR (aortho.py:74-79)."""
    norms = np.linalg.norm(W, axis=0)
    if np.any(norms == 0.0):
        raise OracleBreakdown(f"zero column {int(np.argmin(norms))} entering Pre-CholQR")
    return W / norms


# ---------------------------------------------------------------------------
# Block A-orthonormalisation (aortho.py:89-110)
# ---------------------------------------------------------------------------

def cgs2_project(W, retained, passes=2):
    """Two-pass block classical Gram-Schmidt against cached (Q, AQ) pairs (aortho.py:89-95)."""
    for _ in range(passes):
        coeffs = [aq.T @ W for _, aq in retained]
        for (q, _), c in zip(retained, coeffs):
            W -= q @ c
    return W


def pre_cholqr_block(W, apply_op, breakdown_tol=1e-14):
    """Pre-CholQR then A-CholQR; returns (W', A W') with A W' recomputed (aortho.py:98-110)."""
    W = unit_columns(W)
    W = right_tri_solve(W, small_cholesky(symmetrize(W.T @ W), breakdown_tol))
    AW = apply_op(W)
    W = right_tri_solve(W, small_cholesky(symmetrize(W.T @ AW), breakdown_tol))
    return W, apply_op(W)


# ---------------------------------------------------------------------------
# The engine (solvers.py:147-187, 319-428) + s-step extension
# ---------------------------------------------------------------------------

class OracleStore:
    """Retained (W, AW) pairs with append-before-trim peak accounting (solvers.py:147-187)."""

    def __init__(self, window=None):
        self.window = window
        self.blocks = []
        self.peak = 0
        self.cols = 0

    def append(self, W, AW):
        self.blocks.append((W, AW))
        self.cols += W.shape[1]
        self.peak = max(self.peak, self.cols)
        while self.window is not None and len(self.blocks) > self.window:
            dropped, _ = self.blocks.pop(0)
            self.cols -= dropped.shape[1]

    def clear(self):
        self.blocks = []
        self.cols = 0

    def last(self):
        return self.blocks[-1]

    def concat(self):
        if not self.blocks:
            return np.zeros((0, 0))
        return np.hstack([w for w, _ in self.blocks])


def run_oracle(row_ptr, col_idx, values, b, owner, t, *, method="sre-cg2", s=1,
               tol=1e-8, kmax=None, retention="full", trunc=None, restart_j=None,
               restart_tol=None, switch_tol=None, true_residual_every=50, x0=None,
               on_iteration=None, x_star=None):
    """Unpreconditioned `_run_engine` (solvers.py:319-428) on a CSR operator.

    Returns a dict with the ConvergenceReport fields (solvers.py:126-144) and
    the true residual / relative error that enlarged_solve adds
    (solvers.py:288-291).  `s > 1` selects the s-step extension (DESIGN.md
    section "s-step"): the candidate is [V1, A V1, ..., A^(s-1) V1] where V1
    is split(r) for a fresh store and otherwise the cached product of the
    newest t columns of the previous block.
    """
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col_idx = np.asarray(col_idx, dtype=np.int64)
    values = np.asarray(values, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    owner = np.asarray(owner, dtype=np.int64)
    n = b.shape[0]

    def op(X):
        if X.ndim == 2:
            return csr_spmm(row_ptr, col_idx, values, X)
        return csr_spmv(row_ptr, col_idx, values, X)

    eff_retention = "trunc" if method == "sre-cg" else retention
    window = 2 if method == "sre-cg" else (trunc if retention == "trunc" else None)
    kmax = kmax if kmax is not None else 2 * n

    def build_chain(first):
        if s == 1:
            return first
        cols = [first]
        for _ in range(s - 1):
            cols.append(op(cols[-1]))
        return np.hstack(cols)

    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    r = b - op(x)
    rho0 = float(np.linalg.norm(r))
    history = [rho0]
    store = OracleStore(window)
    restarts, notes, true_checks = [], [], []
    switch_iteration = None
    cur_owner, cur_t = owner, t
    tol1 = 1.0
    best_rho, best_k = rho0, 0
    stagnation_window = max(20, kmax // 10) if eff_retention == "restart" else None
    status = "converged" if rho0 == 0.0 else None

    k = 1
    while status is None and history[-1] > tol * rho0 and k <= kmax:
        if k > 1 and eff_retention == "restart" and k % restart_j == 1:
            store.clear()
            restarts.append(k)
        elif (k > 1 and eff_retention == "restart-tol" and tol1 < restart_tol
              and (not restarts or k > restarts[-1] + 1)):
            store.clear()
            restarts.append(k)

        if switch_tol is not None and switch_iteration is None and k > 1 and tol1 < switch_tol:
            cur_owner, cur_t = halve_owner(cur_owner), cur_t // 2
            switch_iteration = k
            W = build_chain(split_block(cur_owner, cur_t, r))
        elif not store.blocks:
            W = build_chain(split_block(cur_owner, cur_t, r))
        elif method in ("sre-cg2", "sre-cg"):
            prev_aw = store.last()[1]
            W = build_chain(prev_aw[:, prev_aw.shape[1] - cur_t:].copy())
        elif method == "modified-msdo-cg":
            W = split_block(cur_owner, cur_t, r)
        else:  # msdo-cg (solvers.py:378-382)
            prev_w, prev_aw = store.last()
            W = split_block(cur_owner, cur_t, r) + prev_w * (-(prev_aw.T @ r))

        try:
            if store.blocks:
                W = cgs2_project(W, store.blocks)
            W, AW = pre_cholqr_block(W, op)
        except OracleBreakdown as exc:
            status = "breakdown"
            notes.append(f"basis breakdown at iteration {k}: {exc}")
            break
        store.append(W, AW)

        alpha = W.T @ r
        x = x + W @ alpha
        r = r - AW @ alpha
        rho = float(np.linalg.norm(r))
        tol1 = abs(rho - history[-1]) / rho0
        history.append(rho)

        if k % true_residual_every == 0:
            true_checks.append((k, float(np.linalg.norm(b - op(x)))))
        if on_iteration is not None:
            on_iteration({"k": k, "x": x, "r": r, "rho": rho, "tol1": tol1,
                          "store": store, "owner": cur_owner})
        if rho < best_rho:
            best_rho, best_k = rho, k
        elif stagnation_window is not None and k - best_k >= stagnation_window:
            status = "stagnated"
            notes.append(f"no residual decrease over {stagnation_window} iterations")
            break
        k += 1

    if status is None:
        status = "converged" if history[-1] <= tol * rho0 else "maxiter"
    out = {
        "status": status,
        "iterations": len(history) - 1,
        "residual_history": np.array(history),
        "switch_iteration": switch_iteration,
        "restart_iterations": restarts,
        "peak_block_vectors": store.peak,
        "true_residual_checks": true_checks,
        "x": x,
        "notes": notes,
        "true_residual": float(np.linalg.norm(b - op(x))),
    }
    if x_star is not None:
        out["relative_error"] = float(np.linalg.norm(x - x_star) / np.linalg.norm(x_star))
    return out


# ---------------------------------------------------------------------------
# Bounded-memory restatement for the full-size fixtures of configs 4 and 5
# (tests/golden/make_full_golden.py).  Same sequence as run_oracle, with
#  * the sparse product done in row chunks (reduceat segments are per row, so
#    every row's association -- and every output bit -- is unchanged);
#  * A Q_i recomputed from Q_i when the projection needs it instead of cached
#    (the cached block IS op(Q_i), aortho.py:110, so the bits are the same);
#  * in-place / row-chunked forms of the block updates, column scaling and
#    triangular solves (row-independent operations).
# Only the BLAS Gram products keep their whole-block form.  The test
# tests/test_oracle_golden.py::test_lowmem_oracle_matches checks it against
# run_oracle on small problems with many chunks.
# ---------------------------------------------------------------------------

def csr_spmm_chunked(row_ptr, col_idx, values, X, chunk_rows, out=None, threads=None):
    """csr_spmm / csr_spmv over row chunks (bitwise the same as the unchunked forms).
    Chunks are independent, so `threads` > 1 runs them on a thread pool (numpy
    releases the GIL inside the gather / multiply / reduceat loops)."""
    n = row_ptr.shape[0] - 1
    vec = X.ndim == 1
    Y = out if out is not None else np.empty(X.shape)

    def one(a):
        b = min(n, a + chunk_rows)
        lo, hi = int(row_ptr[a]), int(row_ptr[b])
        rp = row_ptr[a:b + 1] - lo
        if vec:
            Y[a:b] = csr_spmv(rp, col_idx[lo:hi], values[lo:hi], X)
            return
        m = X.shape[1]
        scale = values[lo:hi, None]
        ci = col_idx[lo:hi]
        for c0 in range(0, m, COLUMN_SLAB):
            c1 = min(m, c0 + COLUMN_SLAB)
            Y[a:b, c0:c1] = np.add.reduceat(scale * X[ci, c0:c1], rp[:-1], axis=0)

    starts = range(0, n, chunk_rows)
    if threads and threads > 1 and len(starts) > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, starts))
    else:
        for a in starts:
            one(a)
    return Y


def _colnorms_chunked(W, chunk_rows):
    """np.linalg.norm(W, axis=0) without an n x m temporary: the axis-0 reduction
    of a C-ordered block accumulates row after row, so carrying the running sum
    across chunks keeps the association."""
    acc = None
    for a in range(0, W.shape[0], chunk_rows):
        sq = W[a:a + chunk_rows] * W[a:a + chunk_rows]
        acc = np.add.reduce(sq if acc is None else np.vstack([acc[None, :], sq]), axis=0)
    return np.sqrt(acc)


def _tri_solve_inplace(W, R, chunk_rows):
    """W <- W R^-1 row chunk by row chunk (each row solves its own system)."""
    if np.any(np.diag(R) == 0.0):
        raise np.linalg.LinAlgError("singular triangular factor")
    for a in range(0, W.shape[0], chunk_rows):
        W[a:a + chunk_rows] = solve_triangular(R, W[a:a + chunk_rows].T, trans="T", lower=False).T


def run_oracle_lowmem(row_ptr, col_idx, values, b, owner, t, *, method="sre-cg2", s=1, tol=1e-8, kmax=None,
                      retention="trunc", trunc=None, true_residual_every=50, chunk_rows=1 << 18,
                      on_iteration=None, threads=None):
    """run_oracle for unpreconditioned SRE-CG2 / SRE-CG (s >= 1, full or truncated
    retention) holding only the retained Q blocks, the candidate and one scratch
    block: what lets the config-4 (256^3, n x 64) fixture run on a 62 GB host."""
    if method not in ("sre-cg2", "sre-cg") or retention not in ("trunc", "full"):
        raise ValueError("run_oracle_lowmem covers sre-cg2 / sre-cg with trunc or full retention")
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col_idx = np.asarray(col_idx, dtype=np.int64)
    values = np.asarray(values, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    owner = np.asarray(owner, dtype=np.int64)
    n = b.shape[0]
    cr = int(chunk_rows)
    op = lambda X, out=None: csr_spmm_chunked(row_ptr, col_idx, values, X, cr, out, threads)  # noqa: E731
    window = 2 if method == "sre-cg" else (trunc if retention == "trunc" else None)
    kmax = kmax if kmax is not None else 2 * n

    x = np.zeros(n)
    r = b - op(x)
    rho0 = float(np.linalg.norm(r))
    history = [rho0]
    Qs = []  # retained Q blocks (A Q recomputed on use)
    cols, peak = 0, 0
    true_checks, notes = [], []
    status = "converged" if rho0 == 0.0 else None
    prev_aw_tail = None  # newest t columns of A W_{k-1}: the next candidate's first slab
    k = 1
    while status is None and history[-1] > tol * rho0 and k <= kmax:
        m = s * t
        W = np.empty((n, m))
        if not Qs:
            W[:, :t] = split_block(owner, t, r)
        else:
            W[:, :t] = prev_aw_tail
        for i in range(1, s):  # s-step chain (run_oracle.build_chain)
            W[:, i * t:(i + 1) * t] = op(np.ascontiguousarray(W[:, (i - 1) * t:i * t]))
        prev_aw_tail = None
        try:
            for _ in range(2):  # cgs2_project: all coefficients from the same W
                coeffs = []
                for q in Qs:
                    aq = op(q)
                    coeffs.append(aq.T @ W)
                    del aq
                for q, c in zip(Qs, coeffs):
                    for a in range(0, n, cr):
                        W[a:a + cr] -= q[a:a + cr] @ c
            # pre_cholqr_block (aortho.py:98-110)
            norms = _colnorms_chunked(W, cr)
            if np.any(norms == 0.0):
                raise OracleBreakdown(f"zero column {int(np.argmin(norms))} entering Pre-CholQR")
            for a in range(0, n, cr):
                W[a:a + cr] /= norms
            _tri_solve_inplace(W, small_cholesky(symmetrize(W.T @ W)), cr)
            AW = op(W)
            _tri_solve_inplace(W, small_cholesky(symmetrize(W.T @ AW)), cr)
            op(W, out=AW)
        except OracleBreakdown as exc:
            status = "breakdown"
            notes.append(f"basis breakdown at iteration {k}: {exc}")
            break
        Qs.append(W)
        cols += m
        peak = max(peak, cols)
        while window is not None and len(Qs) > window:
            Qs.pop(0)
            cols -= m
        alpha = W.T @ r
        x = x + W @ alpha
        r = r - AW @ alpha
        prev_aw_tail = AW if s == 1 else AW[:, m - t:].copy()
        del AW
        rho = float(np.linalg.norm(r))
        tol1 = abs(rho - history[-1]) / rho0
        history.append(rho)
        if k % true_residual_every == 0:
            true_checks.append((k, float(np.linalg.norm(b - op(x)))))
        if on_iteration is not None:
            on_iteration({"k": k, "rho": rho, "tol1": tol1})
        k += 1
    if status is None:
        status = "converged" if history[-1] <= tol * rho0 else "maxiter"
    return {"status": status, "iterations": len(history) - 1, "residual_history": np.array(history),
            "peak_block_vectors": peak, "true_residual_checks": true_checks, "x": x, "notes": notes,
            "true_residual": float(np.linalg.norm(b - op(x)))}
