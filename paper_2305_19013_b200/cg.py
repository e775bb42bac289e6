"""Classical (optionally block-Jacobi preconditioned) conjugate gradient on the
device: the reference's `cg` (solvers.py:199-258), which `enlarged_solve`
dispatches to for method "cg" (solvers.py:271-272).

Same recurrences and report fields; the products, dot products and updates run
on the sm_100a kernels (operator apply, split-K Gram with m = 1, the fused
x / r update with m = 1, the block-diagonal preconditioner solves), with host
reads of p^T A p, |r| and r^T z every iteration.  Unpreconditioned solves of up to
2^18 rows run the whole loop in one cluster kernel instead (ekcg_cluster_cg,
csrc/cluster_solve.cu): 9 us per iteration at config 1 against 153.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .device import current_stream_ptr, get_device
from .operators import as_operator
from .solvers import ConvergenceReport, SolverConfig, _as_float_vec


class _Dev:
    """Scalar helpers on one stream."""

    def __init__(self, n, device):
        self.n, self.device = n, device
        self.st = current_stream_ptr(device)
        self.chunks_dot = _lib.query("ekcg_gram_chunks", n, 1, 1, 1)
        self.vchunks = _lib.query("ekcg_vec_chunks", n)
        f64 = dict(dtype=torch.float64, device=device)
        self.part = torch.empty(max(self.chunks_dot, self.vchunks), **f64)
        self.tab = torch.empty(1, dtype=torch.int64, device=device)

    def dot(self, x, y, out):
        """out[0] = x . y (deterministic split-K reduction)."""
        self.tab.fill_(x.data_ptr())
        _lib.call("ekcg_gram", self.tab.data_ptr(), 1, 1, 1, y.data_ptr(), 1, 1, self.n, self.part.data_ptr(), None,
                  self.st)
        _lib.call("ekcg_reduce", self.part.data_ptr(), self.chunks_dot, 1, out.data_ptr(), None, self.st)

    def sumsq(self, v, out):
        _lib.call("ekcg_sumsq", v.data_ptr(), self.n, self.part.data_ptr(), None, self.st)
        _lib.call("ekcg_reduce", self.part.data_ptr(), self.vchunks, 1, out.data_ptr(), None, self.st)


def cg(A, b, x0=None, cfg=None, x_star=None, device=None):
    """Classical CG (solvers.py:199-258): returns (x, ConvergenceReport)."""
    cfg = cfg if cfg is not None else SolverConfig(method="cg")
    if cfg.method != "cg":
        raise ValueError(f"cg() called with method {cfg.method!r}; use enlarged_solve")
    cfg.validate()
    n = int(A.n)
    numpy_io = not isinstance(b, torch.Tensor)
    b = _as_float_vec(b, n, "b")
    x0 = _as_float_vec(x0, n, "x0")
    dev = get_device(device if device is not None else (b.device if isinstance(b, torch.Tensor) and b.is_cuda
                                                           else None))
    op = as_operator(A, dev)
    pc = None
    if cfg.preconditioner is not None:
        from .precond import DevicePreconditioner
        F = cfg.preconditioner
        if int(F.n) != n:
            raise ValueError("preconditioner dimension does not match the matrix")
        pc = F if isinstance(F, DevicePreconditioner) else DevicePreconditioner(F, dev)
    kmax = cfg.kmax if cfg.kmax is not None else 2 * n
    f64 = dict(dtype=torch.float64, device=dev)
    h = _Dev(n, dev)
    st = h.st

    bt = torch.as_tensor(b, dtype=torch.float64).to(dev).contiguous()
    x = torch.zeros(n, **f64) if x0 is None else torch.as_tensor(x0, dtype=torch.float64).to(dev).clone()
    r, Ap, z, tmp = (torch.empty(n, **f64) for _ in range(4))
    s = torch.empty(4, **f64)  # [rho^2, p.Ap, r.z, alpha / beta]
    op.apply(x, 1, Ap, 1, 1, None, st)
    _lib.call("ekcg_sub", bt.data_ptr(), Ap.data_ptr(), r.data_ptr(), n, None, st)

    def rnorm():
        h.sumsq(r, s[0:1])
        return float(torch.sqrt(s[0]).item())

    if pc is None and _cluster_cg_ok(op, n, kmax):
        # small problems: the whole loop in one cluster kernel (csrc/cluster_solve.cu), no host reads inside it
        from .operators import StencilOperator
        h.sumsq(r, s[0:1])
        ctrl = torch.zeros(_lib.query("ekcg_ctrl_bytes"), dtype=torch.uint8, device=dev)
        hist = torch.zeros(kmax + 1, **f64)
        _lib.call("ekcg_start", ctrl.data_ptr(), s[0:1].data_ptr(), float(cfg.tol), hist.data_ptr(), st)
        scratch = torch.empty(2 * n, **f64)
        if isinstance(op, StencilOperator):
            desc, rp, ci, vv = op.desc_ref(), None, None, None
        else:
            desc, rp, ci, vv = None, op.row_ptr.data_ptr(), op.col_idx.data_ptr(), op.values.data_ptr()
        _lib.call("ekcg_cluster_cg", desc, rp, ci, vv, n, kmax, x.data_ptr(), r.data_ptr(), scratch.data_ptr(),
                  ctrl.data_ptr(), hist.data_ptr(), st)
        raw = ctrl.cpu().numpy()
        ints, dbl = raw[:32].view(np.int32), raw[32:80].view(np.float64)
        code, k_done = int(ints[1]), int(ints[2])
        if code == 5:
            raise _lib.KernelError("ekcg_cluster_cg refused the matrix: a CSR row holds more than 8 entries")
        history = list(hist[: k_done + 1].cpu().numpy())
        notes = []
        if code == 3:
            status = "breakdown"
            notes.append(f"nonpositive curvature p^T A p = {float(dbl[0]):.3e} at iteration {int(ints[5])}")
        elif code == 0:  # rho0 == 0: the kernel had nothing to do
            status = "converged"
        else:
            status = "converged" if history[-1] <= cfg.tol * history[0] else "maxiter"
        return _finish(op, bt, x, Ap, tmp, h, s, st, n, dev, x_star, numpy_io, status, history, notes)

    def precondition():
        if pc is None:
            return r
        pc.apply(pc.FORWARD, r, 1, tmp, 1, 1, None, st)
        pc.apply(pc.BACKWARD, tmp, 1, z, 1, 1, None, st)
        return z

    rho0 = rnorm()
    history, notes, status = [rho0], [], None
    if rho0 == 0.0:
        status = "converged"
    else:
        zz = precondition()
        p = zz.clone()
        h.dot(r, zz, s[2:3])
        rz = float(s[2].item())
        k = 1
        while history[-1] > cfg.tol * rho0 and k <= kmax:
            op.apply(p, 1, Ap, 1, 1, None, st)
            h.dot(p, Ap, s[1:2])
            pAp = float(s[1].item())
            if pAp <= 0.0:
                status = "breakdown"
                notes.append(f"nonpositive curvature p^T A p = {pAp:.3e} at iteration {k}")
                break
            s[3] = rz / pAp  # alpha, the reference's float division
            # x += alpha p ; r -= alpha Ap ; partial |r|^2 (the m = 1 iterate update)
            _lib.call("ekcg_xr_update", p.data_ptr(), 1, Ap.data_ptr(), 1, s[3:4].data_ptr(), 1, x.data_ptr(),
                      r.data_ptr(), n, h.part.data_ptr(), None, st)
            _lib.call("ekcg_reduce", h.part.data_ptr(), h.vchunks, 1, s[0:1].data_ptr(), None, st)
            history.append(float(torch.sqrt(s[0]).item()))
            zz = precondition()
            h.dot(r, zz, s[2:3])
            rz_new = float(s[2].item())
            s[3] = rz_new / rz  # beta
            rz = rz_new
            # p = z + beta p
            h.tab.fill_(p.data_ptr())
            _lib.call("ekcg_block_update", h.tab.data_ptr(), 1, 1, 1, s[3:4].data_ptr(), zz.data_ptr(), 1,
                      p.data_ptr(), 1, 1, 1.0, 1.0, n, None, st)
            k += 1
        if status is None:
            status = "converged" if history[-1] <= cfg.tol * rho0 else "maxiter"

    return _finish(op, bt, x, Ap, tmp, h, s, st, n, dev, x_star, numpy_io, status, history, notes)


# measured (tools/cluster_cg_time.py): 9 vs 153 us per iteration at n = 10,000, 79 vs 135 at n = 262,144
CLUSTER_CG_MAX_N = 1 << 18


def _cluster_cg_ok(op, n, kmax):
    """The one-kernel cluster CG covers whole-grid stencil operators and CSR matrices with rows of at most
    8 entries, up to CLUSTER_CG_MAX_N rows."""
    from .operators import CsrOperator, StencilOperator
    if n > CLUSTER_CG_MAX_N or kmax + 1 > (1 << 22):
        return False
    if isinstance(op, StencilOperator):
        return True
    if isinstance(op, CsrOperator):
        if not hasattr(op, "_max_row"):
            op._max_row = int((op.row_ptr[1:] - op.row_ptr[:-1]).max().item()) if n else 0
        return op._max_row <= 8
    return False


def _finish(op, bt, x, Ap, tmp, h, s, st, n, dev, x_star, numpy_io, status, history, notes):
    """True residual, relative error and the report (solvers.py:248-258)."""
    op.apply(x, 1, Ap, 1, 1, None, st)
    _lib.call("ekcg_sub", bt.data_ptr(), Ap.data_ptr(), tmp.data_ptr(), n, None, st)
    h.sumsq(tmp, s[0:1])
    true_res = float(torch.sqrt(s[0]).item())
    rel = None
    if x_star is not None:
        xs = torch.as_tensor(x_star, dtype=torch.float64).to(dev)
        rel = float((torch.linalg.vector_norm(x - xs) / torch.linalg.vector_norm(xs)).item())
    x_out = x.cpu().numpy() if numpy_io else x
    rep = ConvergenceReport(status=status, iterations=len(history) - 1, residual_history=np.array(history),
                            peak_block_vectors=0, x=x_out, notes=notes, true_residual=true_res, relative_error=rel)
    return x_out, rep
