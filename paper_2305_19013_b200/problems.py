"""Input side: grid diffusion operators, box partitions, right-hand sides and the
five BASELINE.json configurations (synthetic stand-ins for the paper's
FreeFem++ matrices).

Host-side fixture generation only -- like the reference's generators.py it
runs once per problem and is not part of the accelerated path.  The CSR
assembly reproduces `_diffusion_matrix` (generators.py:25-60) bit for bit;
tests/test_problems.py pins that against hashes of the reference's output.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .linalg import SparseSpdMatrix
from .operators import StencilOperator
from .partition import Partition, contiguous_partition

__all__ = [
    "diffusion_csr",
    "gen_poisson2d",
    "gen_poisson3d",
    "gen_aniso3d",
    "gen_skyscraper",
    "box_owner",
    "box_partition",
    "Problem",
    "make_config",
    "CONFIG_NAMES",
]


def _harmonic(klo, khi):
    # generators.py:45 -- `2.0 * ka * kb / (ka + kb)`, left to right
    return 2.0 * klo * khi / (klo + khi)


def diffusion_csr(shape, kappa, axis_coef=None):
    """CSR of the Dirichlet diffusion stencil for node conductivities `kappa`.

    shape = (nx, ny[, nz]) with x fastest (generators.py:9).  axis_coef scales
    each axis's faces and boundary terms (None = reference operator).
    """
    shape = tuple(int(s) for s in shape)
    dim = len(shape)
    n = int(np.prod(shape))
    K = np.asarray(kappa, dtype=np.float64).reshape(shape[::-1])  # array axes slowest-first
    coef = (1.0,) * dim if axis_coef is None else tuple(float(c) for c in axis_coef)
    coef_slow_first = coef[::-1]

    diag = np.zeros(K.shape)
    faces_lo = []   # per array axis: coefficient to the lower neighbour (0 where absent)
    faces_hi = []
    for ax in range(dim):
        c = coef_slow_first[ax]
        lo = [slice(None)] * dim
        hi = [slice(None)] * dim
        lo[ax] = slice(None, -1)
        hi[ax] = slice(1, None)
        face = _harmonic(K[tuple(lo)], K[tuple(hi)])
        if c != 1.0:
            face = c * face
        f_hi = np.zeros(K.shape)
        f_hi[tuple(lo)] = face
        f_lo = np.zeros(K.shape)
        f_lo[tuple(hi)] = face
        # accumulation order of generators.py:50-53: hi face, lo face, first, last
        diag = diag + f_hi
        diag = diag + f_lo
        for pos in (0, -1):
            side = [slice(None)] * dim
            side[ax] = pos
            bnd = np.zeros(K.shape)
            bnd[tuple(side)] = K[tuple(side)] if c == 1.0 else c * K[tuple(side)]
            diag = diag + bnd
        faces_lo.append(f_lo)
        faces_hi.append(f_hi)

    # row entries in ascending column order: slow-axis lo ... fast-axis lo, diag, fast hi ... slow hi
    strides = [int(np.prod(shape[:dim - 1 - ax])) for ax in range(dim)]  # array-axis strides
    coords = np.indices(K.shape)
    cols_per_slot, vals_per_slot, present = [], [], []
    idx = np.arange(n).reshape(K.shape)
    for ax in range(dim):
        present.append(coords[ax] > 0)
        cols_per_slot.append(idx - strides[ax])
        vals_per_slot.append(-faces_lo[ax])
    present.append(np.ones(K.shape, dtype=bool))
    cols_per_slot.append(idx)
    vals_per_slot.append(diag)
    for ax in reversed(range(dim)):
        present.append(coords[ax] < K.shape[ax] - 1)
        cols_per_slot.append(idx + strides[ax])
        vals_per_slot.append(-faces_hi[ax])
    P = np.stack([p.reshape(-1) for p in present], axis=1)
    C = np.stack([c.reshape(-1) for c in cols_per_slot], axis=1)
    V = np.stack([v.reshape(-1) for v in vals_per_slot], axis=1)
    row_ptr = np.concatenate(([0], np.cumsum(P.sum(axis=1)))).astype(np.int64)
    return SparseSpdMatrix(n, row_ptr, C[P].astype(np.int64), V[P], validate=False)


def _dims(*d):
    for v in d:
        if int(v) < 2:
            raise ValueError(f"grid dimensions must be >= 2, got {d}")
    return tuple(int(v) for v in d)


def gen_poisson2d(nx, ny):
    """5-point Laplacian, Dirichlet (generators.py:70-73)."""
    nx, ny = _dims(nx, ny)
    return diffusion_csr((nx, ny), np.ones(nx * ny))


def gen_poisson3d(nx, ny, nz):
    """7-point Laplacian, Dirichlet (generators.py:76-79)."""
    nx, ny, nz = _dims(nx, ny, nz)
    return diffusion_csr((nx, ny, nz), np.ones(nx * ny * nz))


def gen_aniso3d(nx, ny, nz, layer_contrast):
    """Layered conductivity cycling {1, c, 1/c} in z (generators.py:82-90)."""
    nx, ny, nz = _dims(nx, ny, nz)
    c = float(layer_contrast)
    if c < 1.0:
        raise ValueError("layer_contrast must be >= 1")
    layers = np.array([1.0, c, 1.0 / c])[np.arange(nz) % 3]
    return diffusion_csr((nx, ny, nz), np.repeat(layers, nx * ny))


def gen_skyscraper(nx, ny, nz=None, contrast=1e3):
    """Checkerboard of cells of edge max(1, dim//4); even parity gets `contrast` (generators.py:93-115)."""
    c = float(contrast)
    if c < 1.0:
        raise ValueError("contrast must be >= 1")
    shape = _dims(nx, ny) if nz is None else _dims(nx, ny, nz)
    cell = [np.arange(d) // max(1, d // 4) for d in shape]
    grids = np.meshgrid(*cell[::-1], indexing="ij")  # slowest-first
    parity = sum(grids)
    kappa = np.where(parity % 2 == 0, c, 1.0).reshape(-1)
    return diffusion_csr(shape, kappa)


def box_owner(shape, boxes):
    """Subdomain id bx + Bx*(by + By*bz) with bx = floor(i*Bx/Nx) per axis."""
    shape = tuple(int(s) for s in shape)
    boxes = tuple(int(b) for b in boxes)
    if len(boxes) != len(shape) or any(b < 1 or b > s for b, s in zip(boxes, shape)):
        raise ValueError(f"invalid box decomposition {boxes} for grid {shape}")
    ids = [(np.arange(s) * b) // s for s, b in zip(shape, boxes)]
    owner = np.zeros(shape[::-1], dtype=np.int64)
    mult = 1
    for ax, (bid, b) in enumerate(zip(ids, boxes)):  # x first (fastest)
        sh = [1] * len(shape)
        sh[len(shape) - 1 - ax] = bid.size
        owner = owner + mult * bid.reshape(sh)
        mult *= b
    return owner.reshape(-1)


def box_partition(shape, boxes):
    t = int(np.prod(boxes))
    return Partition.from_owner(box_owner(shape, boxes), t)


# ---------------------------------------------------------------------------
# BASELINE.json configurations
# ---------------------------------------------------------------------------

CONFIG_NAMES = {
    1: "cfg1-srecg-t8-poisson2d-100",
    2: "cfg2-srecg2-t16-poisson3d-64-full",
    3: "cfg3-trunc4-srecg2-t32-skyscraper3d-128",
    4: "cfg4-sstep4-srecg2-t16-aniso3d-256-trunc2",
    5: "cfg5-trunc3-srecg2-t64-tiled2d-8192",
}

FULL_EDGE = {1: 100, 2: 64, 3: 128, 4: 256, 5: 8192}


@dataclass
class Problem:
    name: str
    index: int
    edge: int
    op: StencilOperator | None
    shape: tuple
    kappa_field: np.ndarray | None
    tile: tuple | None
    axis_coef: tuple | None
    partition: Partition
    solver_kwargs: dict
    b: np.ndarray
    x_star: np.ndarray | None
    notes: list = field(default_factory=list)

    @property
    def n(self):
        return int(np.prod(self.shape))

    def node_kappa(self):
        if self.kappa_field is None:
            return np.ones(self.n)
        idx = [np.arange(s) // t for s, t in zip(self.shape, self.tile)]
        f = self.kappa_field
        if len(self.shape) == 2:
            return f[idx[1][:, None], idx[0][None, :]].reshape(-1)
        return f[idx[2][:, None, None], idx[1][None, :, None], idx[0][None, None, :]].reshape(-1)

    def csr(self):
        """Host CSR (reference-generator bits) -- for the oracle and the CSR path."""
        return diffusion_csr(self.shape, self.node_kappa(), self.axis_coef)

    def stencil(self, device=None):
        if self.kappa_field is None:
            return StencilOperator(self.shape, None, None, self.axis_coef, device=device)
        return StencilOperator(self.shape, self.kappa_field, self.tile, self.axis_coef, device=device)


def _rhs_from_solution(csr_or_none, stencil_builder, x_star, prefer_device):
    """b = A x*, bitwise the reference's spmv(A, x*) (linalg.py:133-138)."""
    if prefer_device:
        import torch
        from .device import as_device
        op = stencil_builder()
        xt, back = as_device(x_star)
        y = torch.empty_like(xt)
        op.apply(xt, 1, y, 1, 1)
        return back(y)
    A = csr_or_none()
    # host fixture path (CPU-only test environments, small sizes)
    return np.add.reduceat(A.values * x_star[A.col_idx], A.row_ptr[:-1])


def make_config(index, edge=None, device_rhs=None):
    """Build configuration `index` (1..5) of BASELINE.json at grid edge `edge`
    (default: the full size).  Scaled instances keep the generator, partition
    and seeds, with the coefficient tiles scaled with the grid (cfg3: 8x8 cells
    per plane; cfg5: 16x16-cell tiles)."""
    import torch

    index = int(index)
    full = FULL_EDGE[index]
    N = full if edge is None else int(edge)
    if device_rhs is None:
        device_rhs = torch.cuda.is_available()
    notes = []
    if index == 1:
        shape = (N, N)
        field, tile, coef = None, None, None
        part = contiguous_partition(N * N, 8)
        x_star = np.random.default_rng(0).standard_normal(N * N)
        kw = dict(method="sre-cg", t=8, tol=1e-8)
        b = None
    elif index == 2:
        shape = (N, N, N)
        field, tile, coef = None, None, None
        part = box_partition(shape, (4, 2, 2))
        x_star = np.random.default_rng(1).standard_normal(N ** 3)
        kw = dict(method="sre-cg2", t=16, tol=1e-8, retention="full")
        b = None
    elif index == 3:
        if N % 8:
            raise ValueError("cfg3 edge must be a multiple of 8")
        shape = (N, N, N)
        cell = N // 8
        ty, tx = np.meshgrid(np.arange(8), np.arange(8), indexing="ij")
        field = np.where((tx % 2 == 0) & (ty % 2 == 0), 1000.0, 1.0).reshape(1, 8, 8)
        tile, coef = (cell, cell, N), None
        part = box_partition(shape, (4, 4, 2))
        x_star = None
        b = np.random.default_rng(2).uniform(-1.0, 1.0, N ** 3)
        kw = dict(method="sre-cg2", t=32, tol=1e-8, retention="trunc", trunc=4)
    elif index == 4:
        shape = (N, N, N)
        field, tile, coef = None, None, (1.0, 1.0, 100.0)
        part = box_partition(shape, (4, 2, 2))
        x_star = np.random.default_rng(3).standard_normal(N ** 3)
        kw = dict(method="sre-cg2", t=16, s=4, tol=1e-8, retention="trunc", trunc=2)
        b = None
    elif index == 5:
        if N % 16:
            raise ValueError("cfg5 edge must be a multiple of 16")
        shape = (N, N)
        nt = N // 16
        field = np.exp(np.random.default_rng(4).uniform(np.log(1e-3), np.log(1e3), (nt, nt)))
        tile, coef = (16, 16), None
        part = box_partition(shape, (8, 8))
        x_star = None
        b = np.random.default_rng(5).uniform(-1.0, 1.0, N * N)
        kw = dict(method="sre-cg2", t=64, tol=1e-6, retention="trunc", trunc=3)
    else:
        raise ValueError(f"unknown configuration {index}")

    prob = Problem(CONFIG_NAMES[index] if N == full else f"{CONFIG_NAMES[index]}@{N}", index, N, None,
                   shape, field, tile, coef, part, kw, None, x_star, notes)
    if b is None:
        b = _rhs_from_solution(prob.csr, prob.stencil, x_star, device_rhs)
    prob.b = b
    return prob
