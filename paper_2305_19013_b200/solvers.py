"""Public solver API (mirrors ekcg.solvers, solvers.py:59-292) over the device engine.

`enlarged_solve(A, b, x0, partition, cfg, x_star, on_iteration)` keeps the
reference signature and `ConvergenceReport` fields; `SolverConfig` gains `s`
(s-step depth, default 1 = the reference methods).  The iteration loop runs
on the GPU (engine.py); there is no CPU execution path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "METHODS",
    "RETENTIONS",
    "SolverConfig",
    "ConvergenceReport",
    "BasisStore",
    "enlarged_solve",
]

METHODS = ("cg", "sre-cg2", "sre-cg", "msdo-cg", "modified-msdo-cg")
RETENTIONS = ("full", "trunc", "restart", "restart-tol")
PRECOND_MODES = ("modified", "explicit-hat")
MAX_BLOCK_WIDTH = 64  # s * t limit of the on-device m x m factorizations


@dataclass
class SolverConfig:
    """Method and policy knobs (solvers.py:64-123) plus the s-step depth `s`."""

    method: str = "sre-cg2"
    t: int = 1
    tol: float = 1e-8
    kmax: int | None = None
    retention: str = "full"
    trunc: int | None = None
    restart_j: int | None = None
    restart_tol: float | None = None
    switch_tol: float | None = None
    preconditioner: object = None
    precond_mode: str = "modified"
    true_residual_every: int = 50
    s: int = 1

    def validate(self, partition=None):
        if self.method not in METHODS:
            raise ValueError(f"unknown method {self.method!r}")
        if not (0.0 < self.tol < 1.0):
            raise ValueError("tol must lie in (0, 1)")
        if self.kmax is not None and self.kmax < 1:
            raise ValueError("kmax must be >= 1")
        if self.precond_mode not in PRECOND_MODES:
            raise ValueError(f"unknown precond_mode {self.precond_mode!r}")
        if self.method == "cg":
            return
        if self.retention not in RETENTIONS:
            raise ValueError(f"unknown retention {self.retention!r}")
        if self.retention == "trunc" and (self.trunc is None or self.trunc < 2):
            raise ValueError("trunc retention needs trunc >= 2")
        if self.retention == "restart" and (self.restart_j is None or self.restart_j < 2):
            raise ValueError("restart retention needs restart_j >= 2")
        if self.retention == "restart-tol" and (
                self.restart_tol is None or not (0.0 < self.restart_tol < 1.0)):
            raise ValueError("restart-tol retention needs restart_tol in (0, 1)")
        if self.method == "sre-cg":
            if self.retention == "trunc" and self.trunc != 2:
                raise ValueError(f"sre-cg is the trunc=2 special case; got trunc={self.trunc}")
            if self.retention in ("restart", "restart-tol"):
                raise ValueError("sre-cg fixes the retention to a trunc=2 window")
        if self.t < 1:
            raise ValueError("t must be >= 1")
        if self.switch_tol is not None:
            if not (0.0 < self.switch_tol < 1.0):
                raise ValueError("switch_tol must lie in (0, 1)")
            if self.t % 2 != 0:
                raise ValueError("the half-width switch needs an even t")
        if self.s < 1:
            raise ValueError("s must be >= 1")
        if self.s > 1 and self.method not in ("sre-cg2", "sre-cg"):
            raise ValueError("the s-step variant is defined for sre-cg2 / sre-cg")
        if self.s > 1 and self.preconditioner is not None:
            raise ValueError("the s-step variant is not defined with preconditioning")
        if self.s * self.t > MAX_BLOCK_WIDTH:
            raise ValueError(f"block width s*t = {self.s * self.t} exceeds {MAX_BLOCK_WIDTH}")
        if self.true_residual_every < 1:
            raise ValueError("true_residual_every must be >= 1")
        if partition is not None and partition.t != self.t:
            raise ValueError(f"config t={self.t} does not match partition t={partition.t}")

    def effective_window(self):
        """Retention window in blocks (None = keep everything), solvers.py:119-123."""
        if self.method == "sre-cg":
            return 2
        return self.trunc if self.retention == "trunc" else None


@dataclass
class ConvergenceReport:
    """Outcome of one solve (solvers.py:126-144) plus device throughput fields."""

    status: str
    iterations: int
    residual_history: np.ndarray
    switch_iteration: int | None = None
    restart_iterations: list = field(default_factory=list)
    peak_block_vectors: int = 0
    relative_error: float | None = None
    true_residual: float | None = None
    true_residual_checks: list = field(default_factory=list)
    x: object = None
    notes: list = field(default_factory=list)
    # B200 additions (not in the reference)
    solve_seconds: float | None = None
    iterations_per_second: float | None = None
    model_bytes: float | None = None
    model_flops: float | None = None

    @property
    def converged(self):
        return self.status == "converged"


class BasisStore:
    """Host view of the retained blocks passed to `on_iteration` (solvers.py:147-187).

    Blocks are device tensors; `.blocks` materialises (W, AW) numpy copies
    on first access (testing/diagnostics only).
    """

    def __init__(self, window, device_blocks, peak, to_host=True):
        self.window = window
        self._dev = device_blocks
        self._host = None
        self.peak = peak
        self._to_host = to_host

    @property
    def blocks(self):
        if self._host is None:
            if self._to_host:
                self._host = [(q.cpu().numpy(), aq.cpu().numpy()) for q, aq in self._dev]
            else:
                self._host = [(q.clone(), aq.clone()) for q, aq in self._dev]
        return self._host

    def last(self):
        return self.blocks[-1]

    @property
    def column_count(self):
        return sum(int(q.shape[1]) for q, _ in self._dev)

    def concat(self):
        if not self._dev:
            return np.zeros((0, 0))
        if self._to_host:
            return np.hstack([w for w, _ in self.blocks])
        import torch
        return torch.hstack([w for w, _ in self.blocks])


def _as_float_vec(v, n, name, device=None):
    """Validation of b / x0 (solvers.py:190-196), for numpy or torch input.  With a device, host
    input is uploaded first and checked there (a 537 MB host scan costs ~60 ms, the device one ~1)."""
    import torch
    if v is None:
        return None
    if not isinstance(v, torch.Tensor):
        arr = np.asarray(v, dtype=np.float64)
        if arr.shape != (n,):
            raise ValueError(f"{name} must have length {n}, got shape {arr.shape}")
        if device is None:
            if not np.all(np.isfinite(arr)):
                raise ValueError(f"{name} must be finite")
            return arr
        v = torch.from_numpy(np.ascontiguousarray(arr)).to(device)
    if tuple(v.shape) != (n,):
        raise ValueError(f"{name} must have length {n}, got shape {tuple(v.shape)}")
    if not bool(torch.all(torch.isfinite(v))):
        raise ValueError(f"{name} must be finite")
    return v


def _solve_explicit_hat(A, b, x0, partition, cfg, x_star, on_iteration, device):
    """Plain engine on L^-1 A L^-T, x = L^-T x_hat (solvers.py:295-316), all on the device."""
    from dataclasses import replace

    import torch

    from .device import as_device
    from .engine import DeviceEngine
    from .operators import HatOperator, as_operator
    from .precond import DevicePreconditioner, backward_solve, forward_solve, mult_lt

    op = as_operator(A, device)
    F = cfg.preconditioner
    pc = F if isinstance(F, DevicePreconditioner) else DevicePreconditioner(F, op.device)
    b_hat = forward_solve(pc, b)
    x0_hat = None if x0 is None else mult_lt(pc, x0)
    engine = DeviceEngine(HatOperator(op, pc), partition, replace(cfg, preconditioner=None), device=device)
    engine.norm_pc = pc
    x_hat, rep = engine.solve(b_hat, x0_hat, on_iteration=on_iteration)
    x = backward_solve(pc, x_hat)
    xt, _ = as_device(x, device=op.device)
    bt, _ = as_device(b, device=op.device)
    ax = torch.empty_like(xt)
    op.apply(xt, 1, ax, 1, 1)
    rep.x = x
    rep.true_residual = float(torch.linalg.vector_norm(bt - ax).item())
    if x_star is not None:
        xs, _ = as_device(x_star, device=op.device)
        rep.relative_error = float((torch.linalg.vector_norm(xt - xs) / torch.linalg.vector_norm(xs)).item())
    return x, rep


def enlarged_solve(A, b, x0=None, partition=None, cfg=None, x_star=None, on_iteration=None,
                   device=None):
    """Run one enlarged-CG method on the GPU (solvers.py:261-292).

    A: SparseSpdMatrix (or any CSR object with n/row_ptr/col_idx/values), or
       an operators.StencilOperator.  b, x0, x_star: numpy or torch.
    Returns (x, ConvergenceReport); x matches b's array type (numpy in,
    numpy out; CUDA tensor in, CUDA tensor out).
    """
    from .engine import DeviceEngine

    cfg = cfg if cfg is not None else SolverConfig()
    if cfg.method == "cg":  # solvers.py:271-272
        from .cg import cg
        return cg(A, b, x0=x0, cfg=cfg, x_star=x_star, device=device)
    if partition is None:
        raise ValueError("enlarged methods need a partition")
    cfg.validate(partition)
    from .partition import Partition
    if not isinstance(partition, Partition):  # e.g. an ekcg.Partition: adopt its owner map
        partition = Partition.from_owner(np.asarray(partition.owner()), partition.t)
    n = int(A.n)
    if partition.n != n:
        raise ValueError(f"partition covers {partition.n} indices, matrix has {n}")
    import torch
    from .device import get_device
    numpy_io = not isinstance(b, torch.Tensor)
    F = cfg.preconditioner
    # host input is validated on the device it is uploaded to (no GPU: the host check, then the engine raises)
    dev = (get_device(device) if torch.cuda.is_available() and (F is None or cfg.precond_mode != "explicit-hat")
           else None)
    b = _as_float_vec(b, n, "b", dev)
    x0 = _as_float_vec(x0, n, "x0", dev)
    if F is not None and int(F.n) != n:
        raise ValueError("preconditioner dimension does not match the matrix")
    if F is not None and cfg.precond_mode == "explicit-hat":
        return _solve_explicit_hat(A, b, x0, partition, cfg, x_star, on_iteration, device)
    import torch.distributed as tdist
    from .operators import StencilOperator
    sharded = (tdist.is_available() and tdist.is_initialized() and tdist.get_world_size() > 1
               and F is None and cfg.method in ("sre-cg2", "sre-cg") and cfg.switch_tol is None
               and on_iteration is None  # callbacks see whole blocks: the single-GPU engine serves them
               and (isinstance(A, StencilOperator) or hasattr(A, "row_ptr") or hasattr(A, "host")))
    if sharded:  # one process per GPU, rows split across ranks
        from .sharded import ShardedEngine
        engine = ShardedEngine(A, partition, cfg, device=device)
    else:
        engine = DeviceEngine(A, partition, cfg, device=device)
    return engine.solve(b, x0, x_star=x_star, on_iteration=on_iteration, numpy_io=numpy_io)
