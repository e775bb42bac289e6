"""CSR matrices with an exact grid-stencil pattern are applied in stencil form
(`StencilOperator.from_csr`, operators.DETECT_GRID): the values go unchanged into the per-node
coefficient table the plane-march / fused kernels read, so every product is bitwise the CSR product
(the reference's spmm, linalg.py:141-152) and a CSR-form solve is bitwise the stencil-form solve."""

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.grid_detect]

import paper_2305_19013_b200 as pk
from paper_2305_19013_b200 import operators
from paper_2305_19013_b200.engine import DeviceEngine
from paper_2305_19013_b200.operators import CsrOperator, StencilOperator, as_operator
from paper_2305_19013_b200.problems import make_config
from paper_2305_19013_b200.solvers import SolverConfig


def _bits(a):
    return np.ascontiguousarray(a).view(np.int64)


@pytest.mark.parametrize("idx,edge,m", [(1, 40, 8), (2, 12, 16), (3, 16, 32), (5, 64, 64), (4, 10, 16), (3, 32, 5),
                                        (1, 100, 1)])
def test_detected_grid_operator_is_bitwise_the_csr_product(idx, edge, m):
    prob = make_config(idx, edge)
    A = prob.csr()
    assert operators.DETECT_GRID
    op = as_operator(A)
    assert isinstance(op, StencilOperator) and op.from_matrix and op.n == prob.n
    assert op.shape == tuple(prob.stencil().shape)
    csr = CsrOperator(A)
    rng = np.random.default_rng(idx)
    X = torch.as_tensor(rng.standard_normal((prob.n, m)), device="cuda")
    X[rng.integers(0, prob.n, 50)] = 0.0  # exact zeros: signed-zero association
    Y1, Y2 = torch.empty_like(X), torch.empty_like(X)
    op.apply(X, m, Y1, m, m)
    csr.apply(X, m, Y2, m, m)
    assert np.array_equal(_bits(Y1.cpu().numpy()), _bits(Y2.cpu().numpy()))
    # the public product goes through the same dispatch
    assert np.array_equal(_bits(pk.spmm(A, X.cpu().numpy())), _bits(Y2.cpu().numpy()))


def test_patterns_that_are_not_a_grid_stay_csr():
    rng = np.random.default_rng(0)
    prob = make_config(2, 8)
    A = prob.csr()
    rp, ci, vals = A.row_ptr.copy(), A.col_idx.copy(), A.values.copy()
    # (a) a symmetric permutation of the grid matrix
    n = A.n
    perm = rng.permutation(n)
    dense = pk.SparseSpdMatrix(n, rp, ci, vals).to_dense()[np.ix_(perm, perm)]
    r, c = np.nonzero(dense)
    P = pk.SparseSpdMatrix.from_coo(n, r, c, dense[r, c])
    assert isinstance(as_operator(P), CsrOperator)
    # (b) one off-diagonal pair dropped (a sparser pattern)
    d2 = pk.SparseSpdMatrix(n, rp, ci, vals).to_dense()
    d2[5, 6] = d2[6, 5] = 0.0
    r, c = np.nonzero(d2)
    assert isinstance(as_operator(pk.SparseSpdMatrix.from_coo(n, r, c, d2[r, c])), CsrOperator)
    # (c) an extra entry (a wider pattern)
    d3 = pk.SparseSpdMatrix(n, rp, ci, vals).to_dense()
    d3[0, 17] = d3[17, 0] = -0.01
    r, c = np.nonzero(d3)
    assert isinstance(as_operator(pk.SparseSpdMatrix.from_coo(n, r, c, d3[r, c])), CsrOperator)
    # (d) a tridiagonal (1-D) matrix, and the identity
    T = np.diag(np.full(30, 2.0)) + np.diag(np.full(29, -1.0), 1) + np.diag(np.full(29, -1.0), -1)
    r, c = np.nonzero(T)
    assert isinstance(as_operator(pk.SparseSpdMatrix.from_coo(30, r, c, T[r, c])), CsrOperator)
    eye = pk.SparseSpdMatrix(12, np.arange(13), np.arange(12), np.ones(12))
    assert isinstance(as_operator(eye), CsrOperator)
    # products of the fallbacks are still the reference's
    X = rng.standard_normal((n, 3))
    assert np.allclose(pk.spmm(P, X), dense @ X, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("idx,edge,over", [(2, 12, {}), (3, 16, {"kmax": 40}), (1, 64, {}), (5, 64, {"kmax": 30})])
def test_csr_form_solve_equals_stencil_form_bitwise(idx, edge, over):
    """With detection on, a reference-facing CSR solve runs the same kernels as the matrix-free form."""
    prob = make_config(idx, edge)
    cfg = SolverConfig(**dict(prob.solver_kwargs, **over))
    xa, a = pk.enlarged_solve(prob.csr(), prob.b, partition=prob.partition, cfg=cfg)
    xb, b = pk.enlarged_solve(prob.stencil(), prob.b, partition=prob.partition, cfg=cfg)
    assert a.status == b.status and a.iterations == b.iterations
    assert np.array_equal(a.residual_history, b.residual_history)
    assert np.array_equal(xa, xb)


def test_detection_off_keeps_the_csr_kernels(monkeypatch):
    prob = make_config(2, 8)
    monkeypatch.setattr(operators, "DETECT_GRID", False)
    assert isinstance(as_operator(prob.csr()), CsrOperator)
    eng = DeviceEngine(prob.csr(), prob.partition, SolverConfig(**prob.solver_kwargs))
    assert isinstance(eng.op, CsrOperator)
