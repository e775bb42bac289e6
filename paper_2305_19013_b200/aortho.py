"""Block A-orthonormalisation on the device: the public functions of the
reference's aortho module (aortho.py:25-71), built on the same sm_100a kernels
the engine uses (split-K DMMA Gram, DMMA block update, device Cholesky, CSR /
stencil SpMM).  numpy in -> numpy out; CUDA tensors stay on the device.

The solver itself does not call these (it runs the fused in-loop forms in
engine.py); they are the test-facing surface a caller of `ekcg` may use.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .device import as_device, current_stream_ptr
from .linalg import Breakdown, _aligned, _ptr_table, cholesky_small, gram, spmm, trsm_right_inv

__all__ = ["a_orthogonalize_against", "a_cholqr", "pre_cholqr"]


def _sym(G):
    return 0.5 * (G + G.T)


def _sub_product(W, Q, C):
    """W - Q C on the device (ekcg_block_update, one block of width k)."""
    n, m = W.shape
    k = Q.shape[1]
    out = torch.empty_like(W)
    if n:
        Qc = _aligned(Q.contiguous())
        tab = _ptr_table(Qc)
        _lib.call("ekcg_block_update", tab.data_ptr(), k, 1, k, C.contiguous().data_ptr(), W.data_ptr(), m,
                  out.data_ptr(), m, m, 1.0, -1.0, n, None, current_stream_ptr(W.device))
    return out


def a_orthogonalize_against(A, W, Q, aq=None, passes=2):
    """`passes` rounds of W <- W - Q (Q^T A W) against an A-orthonormal Q
    (aortho.py:25-44); with `aq` (= A Q) the coefficients are aq^T W,
    otherwise Q^T (A W) with A W recomputed per pass.  Empty Q: W unchanged."""
    Wt, back = as_device(W)
    Wt = Wt.to(torch.float64).clone().contiguous()
    if Q is None:
        return back(Wt)
    Qt, _ = as_device(Q, device=Wt.device)
    if Qt.dim() != 2 or Qt.shape[1] == 0:
        return back(Wt)
    if Qt.shape[0] != Wt.shape[0] or Qt.shape[0] != A.n:
        raise ValueError("row-count mismatch between A, W and Q")
    Qt = Qt.contiguous()
    AQ = None if aq is None else as_device(aq, device=Wt.device)[0].contiguous()
    for _ in range(passes):
        C = gram(AQ, Wt) if AQ is not None else gram(Qt, spmm(A, Wt))
        Wt = _sub_product(Wt, Qt, C)
    return back(Wt)


def a_cholqr(A, W, breakdown_tol=1e-14):
    """W R^-1 with R = chol(sym(W^T A W)), so W'^T A W' = I (aortho.py:47-57);
    raises Breakdown on numerical rank deficiency in the A-inner product."""
    Wt, back = as_device(W)
    Wt = Wt.to(torch.float64).contiguous()
    G = _sym(gram(Wt, spmm(A, Wt)))
    R = cholesky_small(G, breakdown_tol)
    return back(trsm_right_inv(Wt, R))


def _scale_columns(W):
    """Columns to unit 2-norm; a zero column raises Breakdown (aortho.py:74-79)."""
    norms = torch.linalg.vector_norm(W, dim=0)
    if bool(torch.any(norms == 0.0)):
        dead = int(torch.argmin(norms).item())
        raise Breakdown(f"zero column {dead} entering Pre-CholQR")
    return W / norms


def pre_cholqr(A, W, breakdown_tol=1e-14):
    """Unit-norm columns, Euclidean CholQR, then A-CholQR (aortho.py:60-71)."""
    Wt, back = as_device(W)
    Wt = _scale_columns(Wt.to(torch.float64).contiguous())
    R0 = cholesky_small(_sym(gram(Wt, Wt)), breakdown_tol)
    return back(a_cholqr(A, trsm_right_inv(Wt, R0), breakdown_tol))
