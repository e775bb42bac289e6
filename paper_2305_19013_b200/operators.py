"""Device operators A: CSR SpMM and the structured-grid stencil (the `op` seam of
`_run_engine`, solvers.py:285-286,319).

Both apply Y = A X to row-major blocks with arbitrary row strides, so the
s-step chain can multiply column slabs of one n x (s*t) block in place.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .device import current_stream_ptr, get_device


EKCG_COEF_STRIDE = {2: 6, 3: 8}


def _ptr(x):
    return x if isinstance(x, int) else x.data_ptr()


class CsrOperator:
    """General SPD matrix in CSR; bit-exact with the reference spmm/spmv."""

    kind = "csr"

    def __init__(self, A, device=None):
        self.device = get_device(device)
        self.n = int(A.n)
        if hasattr(A, "device_arrays"):
            self.row_ptr, self.col_idx, self.values = A.device_arrays(self.device)
        else:  # duck-typed reference matrix (ekcg.SparseSpdMatrix)
            self.row_ptr = torch.from_numpy(np.ascontiguousarray(A.row_ptr, dtype=np.int64)).to(self.device)
            self.col_idx = torch.from_numpy(np.ascontiguousarray(A.col_idx, dtype=np.int32)).to(self.device)
            self.values = torch.from_numpy(np.ascontiguousarray(A.values, dtype=np.float64)).to(self.device)
        self.nnz = int(self.col_idx.numel())
        self.host = A

    def matrix_bytes(self):
        """Bytes of A streamed per application (int64 row_ptr, int32 col, f64 val)."""
        return 8 * (self.n + 1) + 12 * self.nnz

    def apply(self, X, ldx, Y, ldy, m, live=None, stream=None):
        st = current_stream_ptr(self.device) if stream is None else stream
        _lib.call("ekcg_spmm_csr", self.row_ptr.data_ptr(), self.col_idx.data_ptr(), self.values.data_ptr(),
                  _ptr(X), ldx, _ptr(Y), ldy, self.n, m, live, st)

    def apply_rows(self, r0, r1, X, ldx, Y, ldy, m, live=None, stream=None):
        """Rows [r0, r1) of Y = A X (Y points at row 0): the row pointers keep
        addressing the full column / value arrays, so a sub-range is a pointer shift."""
        if r1 <= r0:
            return
        st = current_stream_ptr(self.device) if stream is None else stream
        _lib.call("ekcg_spmm_csr", self.row_ptr.data_ptr() + 8 * r0, self.col_idx.data_ptr(),
                  self.values.data_ptr(), _ptr(X), ldx, _ptr(Y) + 8 * r0 * ldy, ldy, r1 - r0, m, live, st)


class StencilOperator:
    """`_diffusion_matrix(shape, kappa)` (generators.py:25-60) applied matrix-free.

    shape: (nx, ny) or (nx, ny, nz), x fastest.
    kappa: None / scalar (constant), or a tile field `field` of shape
           (fz, fy, fx) / (fy, fx) with tile edge `tile` = (tx, ty[, tz]);
           tile (1,1,1) with a full-size field is a node-by-node kappa.
    axis_coef: per-axis multipliers (cx, cy[, cz]) on face and boundary
           coefficients; all ones reproduces the reference generator exactly.
    """

    kind = "stencil"

    def __init__(self, shape, kappa=None, tile=None, axis_coef=None, device=None):
        self.device = get_device(device)
        shape = tuple(int(s) for s in shape)
        if len(shape) not in (2, 3) or min(shape) < 2:
            raise ValueError(f"grid dimensions must be >= 2, got {shape}")
        self.shape = shape
        self.dim = len(shape)
        self.n = int(np.prod(shape))
        coef = tuple(float(c) for c in (axis_coef or (1.0,) * self.dim))
        if len(coef) != self.dim:
            raise ValueError("axis_coef needs one entry per grid axis")
        self.axis_coef = coef
        desc = _lib.EkcgStencil()
        desc.dim = self.dim
        desc.nx, desc.ny = shape[0], shape[1]
        desc.nz = shape[2] if self.dim == 3 else 1
        desc.cx, desc.cy = coef[0], coef[1]
        desc.cz = coef[2] if self.dim == 3 else 1.0
        self.field = None
        if kappa is None or np.isscalar(kappa):
            desc.kfield = None
            desc.kconst = 1.0 if kappa is None else float(kappa)
            desc.tx = desc.ty = desc.tz = 1
            desc.fx = desc.fy = 1
            self.field_host = None
        else:
            field = np.ascontiguousarray(np.asarray(kappa, dtype=np.float64))
            tile = tuple(int(v) for v in (tile or (1,) * self.dim))
            if len(tile) != self.dim:
                raise ValueError("tile needs one entry per grid axis")
            need = tuple(-(-s // t) for s, t in zip(shape, tile))  # tiles per axis (x, y[, z])
            if field.shape != need[::-1]:
                if field.size == self.n and all(t == 1 for t in tile):
                    field = field.reshape(shape[::-1])
                else:
                    raise ValueError(f"kappa field shape {field.shape} != tiles {need[::-1]}")
            if not np.all(np.isfinite(field)) or np.any(field <= 0.0):
                raise ValueError("kappa must be finite and positive")
            self.field_host = field
            self.field = torch.from_numpy(field.reshape(-1)).to(self.device)
            desc.kfield = self.field.data_ptr()
            # harmonic mean of each tile with itself, 2*k*k/(k+k) left to right
            # (generators.py:45 with ka = kb): same-tile faces skip the division
            self.kself = torch.from_numpy(np.ascontiguousarray(2.0 * field * field / (field + field)).reshape(-1)).to(
                self.device)
            desc.kself = self.kself.data_ptr()
            # faces between a tile and its +x / +y / +z neighbour tile (generators.py:45 on the
            # host: c * ((2 k_lo k_hi) / (k_lo + k_hi)), left to right): cross-tile faces load
            # them instead of dividing on the device
            f3 = field if self.dim == 3 else field[None]
            cz = coef[2] if self.dim == 3 else 1.0
            self.hcross = []
            for axis, c in ((2, coef[0]), (1, coef[1]), (0, cz)):
                h = np.zeros_like(f3)
                lo = [slice(None)] * 3
                hi = [slice(None)] * 3
                lo[axis], hi[axis] = slice(0, -1), slice(1, None)
                klo, khi = f3[tuple(lo)], f3[tuple(hi)]
                h[tuple(lo)] = c * (2.0 * klo * khi / (klo + khi))
                self.hcross.append(torch.from_numpy(np.ascontiguousarray(h).reshape(-1)).to(self.device))
            desc.hx, desc.hy, desc.hz = (t.data_ptr() for t in self.hcross)
            desc.tx, desc.ty = tile[0], tile[1]
            desc.tz = tile[2] if self.dim == 3 else 1
            desc.fx, desc.fy = need[0], need[1]
            desc.kconst = 0.0
        self.tile = (desc.tx, desc.ty, desc.tz)
        self._desc = desc
        self.coef = None
        if self.field is not None and self.dim == 3:
            # per-node coefficient rows, built once on the device by the kernels' own arithmetic
            # (ekcg_stencil_coefs): every later application loads a row instead of recomputing the
            # tile lookups and faces of each node in each column chunk.  Measured: config-3 march
            # 0.363 -> 0.326 ms; in 2-D (config 5) the extra 48 B per node made it 1.7 % slower
            # (tools/probe_stencil.py), so 2-D fields keep the on-the-fly coefficients.
            stride = 8 if self.dim == 3 else 6
            self.coef = torch.empty(self.n * stride, dtype=torch.float64, device=self.device)
            _lib.call("ekcg_stencil_coefs", ctypes.byref(desc), self.coef.data_ptr(),
                      current_stream_ptr(self.device))
            desc.coef = self.coef.data_ptr()

    @classmethod
    def from_csr(cls, csr):
        """The grid-stencil form of a CSR matrix whose sparsity pattern is exactly the 5- / 7-point
        pattern of an nx x ny (x nz) grid in x-fastest order (what `_diffusion_matrix`,
        `gen_poisson2d/3d` and any finite-volume assembly on a box grid produce), or None.

        The values go, unchanged, into the per-node coefficient table the plane-march and fused
        stencil kernels already read (EkcgStencil.coef: slot order z-, y-, x-, diag, x+, y+, z+), so
        every product is bitwise the CSR product (same entries, same order, same association) while
        each X row is staged once through shared memory instead of gathered up to 7 times from L2,
        and the fused m <= 16 kernels and the matrix-free cluster path apply.  The check is exact:
        row pointers and every column index must equal the grid pattern's (done on the device)."""
        n = int(csr.n)
        rp, ci, vals = csr.row_ptr, csr.col_idx, csr.values
        if n < 4 or rp.numel() != n + 1:
            return None
        dev = rp.device
        head = rp[:2].cpu().tolist()
        cnt0 = head[1] - head[0]
        if head[0] != 0 or cnt0 not in (3, 4):
            return None
        c0 = ci[:cnt0].cpu().tolist()
        if c0[0] != 0 or c0[1] != 1 or c0[2] < 2:
            return None
        nx = int(c0[2])
        if cnt0 == 4:
            nxy = int(c0[3])
            if nxy % nx or n % nxy:
                return None
            ny, nz, dim = nxy // nx, n // nxy, 3
        else:
            if n % nx:
                return None
            ny, nz, dim, nxy = n // nx, 1, 2, n
        if ny < 2 or (dim == 3 and nz < 2) or n >= (1 << 31):
            return None
        i = torch.arange(n, dtype=torch.int64, device=dev)
        x, y, z = i % nx, (i // nx) % ny, i // nxy
        true = torch.ones(n, dtype=torch.bool, device=dev)
        slots = [(-nxy, z > 0), (-nx, y > 0), (-1, x > 0), (0, true), (1, x < nx - 1), (nx, y < ny - 1),
                 (nxy, z < nz - 1)]
        if dim == 2:
            slots = slots[1:6]
        count = torch.zeros(n, dtype=torch.int64, device=dev)
        for _, present in slots:
            count += present
        expect_rp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        torch.cumsum(count, 0, out=expect_rp[1:])
        nnz = int(ci.numel())
        # one verdict, read back once: row pointers equal, and every present slot holds the grid neighbour
        ok = (expect_rp == rp.to(torch.int64)).all() & (expect_rp[-1] == nnz)
        stride = 8 if dim == 3 else 6
        table = torch.zeros(n, stride, dtype=torch.float64, device=dev)
        pos = expect_rp[:-1].clone()
        last = max(nnz - 1, 0)
        for slot, (off, present) in enumerate(slots):
            at = pos.clamp(max=last)
            ok = ok & torch.where(present, ci[at].to(torch.int64) == i + off, true).all()
            table[:, slot] = torch.where(present, vals[at], table[:, slot])
            pos += present
        if not bool(ok):
            return None
        op = cls.__new__(cls)
        op.device = dev
        op.shape = (nx, ny) if dim == 2 else (nx, ny, nz)
        op.dim, op.n = dim, n
        op.axis_coef = (1.0,) * dim
        op.field = op.field_host = None
        op.coef = table.reshape(-1)
        op.tile = (1, 1, 1)
        op.nnz = int(ci.numel())
        op.host = getattr(csr, "host", None)
        op.from_matrix = True
        desc = _lib.EkcgStencil()
        desc.dim, desc.nx, desc.ny, desc.nz = dim, nx, ny, nz
        desc.cx = desc.cy = desc.cz = 1.0
        desc.kfield = op.coef.data_ptr()  # non-null marks a variable-coefficient operator; never read:
        desc.coef = op.coef.data_ptr()    # every kernel takes a node's row from the table
        desc.tx = desc.ty = desc.tz = 1
        desc.fx, desc.fy = nx, ny
        desc.kconst = 0.0
        op._desc = desc
        return op

    def matrix_bytes(self):
        """M_A of the SURVEY 8(d) traffic model: 0 for constant kappa, 8 n (a node-kappa array) for a
        kappa field.  The kernels actually stream the per-node coefficient table (48 n / 64 n bytes
        in 2-D / 3-D); DESIGN.md section 3 and the ncu traffic columns account for it."""
        if getattr(self, "from_matrix", False):  # the coefficient table of a CSR matrix in grid form
            return 8 * EKCG_COEF_STRIDE[self.dim] * self.n
        return 0 if self.field is None else 8 * self.n

    def node_kappa(self):
        """Full node-kappa array (host), x fastest."""
        if getattr(self, "from_matrix", False):
            raise ValueError("an operator built from a CSR matrix has no kappa field")
        if self.field_host is None:
            return np.full(self.n, self._desc.kconst)
        f = self.field_host
        idx = [np.arange(s) // t for s, t in zip(self.shape, self.tile)]
        if self.dim == 2:
            return f[idx[1][:, None], idx[0][None, :]].reshape(-1)
        return f[idx[2][:, None, None], idx[1][None, :, None], idx[0][None, None, :]].reshape(-1)

    def to_csr(self):
        """Host CSR of the same operator (bitwise the reference generator's)."""
        from .problems import diffusion_csr
        return diffusion_csr(self.shape, self.node_kappa(), self.axis_coef)

    def desc_ref(self):
        return ctypes.byref(self._desc)

    def apply(self, X, ldx, Y, ldy, m, live=None, stream=None):
        st = current_stream_ptr(self.device) if stream is None else stream
        _lib.call("ekcg_spmm_stencil", ctypes.byref(self._desc), _ptr(X), ldx, _ptr(Y), ldy, m, live, st)


# CSR matrices with an exact grid-stencil pattern are applied in stencil form (StencilOperator.from_csr):
# bitwise the same products, stencil-kernel speed.  False keeps every CSR matrix on the CSR kernels.
DETECT_GRID = True


def as_operator(A, device=None):
    if isinstance(A, (CsrOperator, StencilOperator, HatOperator)):
        return A
    if hasattr(A, "row_ptr") and hasattr(A, "col_idx") and hasattr(A, "values"):
        dev = get_device(device)
        # the operator is cached on the host matrix (immutable by contract: SparseSpdMatrix keeps its
        # device arrays in `_dev` the same way)
        cache = getattr(A, "_dev", None)
        if not isinstance(cache, dict):
            cache = getattr(A, "_ekcg_ops", None)
            if cache is None:
                cache = {}
                try:
                    setattr(A, "_ekcg_ops", cache)
                except AttributeError:
                    pass
        key = ("operator", str(dev), bool(DETECT_GRID))
        if key in cache:
            return cache[key]
        op = CsrOperator(A, dev)
        if DETECT_GRID:
            grid = StencilOperator.from_csr(op)
            if grid is not None:
                op = grid
        cache[key] = op
        return op
    raise TypeError(f"unsupported operator type {type(A).__name__}")


class HatOperator:
    """L^-1 A L^-T for the explicit-hat preconditioned mode (solvers.py:295-316)."""

    kind = "hat"

    def __init__(self, op, pc):
        self.op, self.pc = op, pc
        self.n = op.n
        self.device = op.device
        self.nnz = op.nnz if hasattr(op, "nnz") else None
        self._tmp = {}

    def matrix_bytes(self):
        return self.op.matrix_bytes()

    def _scratch(self, m):
        if m not in self._tmp:
            f64 = dict(dtype=torch.float64, device=self.device)
            self._tmp[m] = (torch.empty(self.n * m, **f64), torch.empty(self.n * m, **f64))
        return self._tmp[m]

    def apply(self, X, ldx, Y, ldy, m, live=None, stream=None):
        t1, t2 = self._scratch(m)
        pc = self.pc
        pc.apply(pc.BACKWARD, _ptr(X), ldx, t1.data_ptr(), m, m, live, stream)
        self.op.apply(t1, m, t2, m, m, live, stream)
        pc.apply(pc.FORWARD, t2.data_ptr(), m, _ptr(Y), ldy, m, live, stream)
