"""The public A-orthonormalisation functions (aortho.py:25-71) on the device:
invariants the reference's own aortho tests check, plus agreement with the
oracle restatement (oracle/ekcg_oracle.py) on the same inputs."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2305_19013_b200 as pk
from oracle import ekcg_oracle as orc


def spd_csr(n, rng, lo=1.0, hi=10.0):
    """Dense SPD matrix with a spectrum in [lo, hi], stored as CSR (and dense)."""
    U, _ = np.linalg.qr(rng.standard_normal((n, n)))
    D = (U * np.linspace(lo, hi, n)) @ U.T
    D = 0.5 * (D + D.T)
    rows, cols = np.nonzero(np.ones((n, n)))
    return pk.SparseSpdMatrix.from_coo(n, rows, cols, D[rows, cols]), D


def eye_csr(n):
    i = np.arange(n)
    return pk.SparseSpdMatrix.from_coo(n, i, i, np.ones(n))


def a_err(W, D):
    return float(np.max(np.abs(W.T @ D @ W - np.eye(W.shape[1]))))


@pytest.fixture
def rng():
    return np.random.default_rng(2305)


def test_orthogonalize_empty_basis_is_identity(rng):
    A, W = eye_csr(7), rng.standard_normal((7, 3))
    assert np.array_equal(pk.a_orthogonalize_against(A, W, np.zeros((7, 0))), W)
    assert np.array_equal(pk.a_orthogonalize_against(A, W, None), W)


def test_orthogonalize_removes_components_in_span(rng):
    A, D = spd_csr(12, rng)
    Q = pk.a_cholqr(A, rng.standard_normal((12, 3)))
    W = Q @ rng.standard_normal((3, 2))
    assert np.linalg.norm(pk.a_orthogonalize_against(A, W, Q)) <= 1e-12 * np.linalg.norm(W)


def test_orthogonalize_two_pass_formula(rng):
    A = eye_csr(9)
    Q = np.eye(9)[:, [1, 4, 6]]
    W = rng.standard_normal((9, 4))
    ref = W.copy()
    for _ in range(2):
        ref = ref - Q @ (Q.T @ ref)
    np.testing.assert_allclose(pk.a_orthogonalize_against(A, W, Q), ref, rtol=1e-13, atol=1e-13)


def test_orthogonalize_cached_product_and_idempotence(rng):
    A, D = spd_csr(11, rng)
    Q = pk.a_cholqr(A, rng.standard_normal((11, 3)))
    W = rng.standard_normal((11, 2))
    plain = pk.a_orthogonalize_against(A, W, Q)
    cached = pk.a_orthogonalize_against(A, W, Q, aq=pk.spmm(A, Q))
    np.testing.assert_allclose(cached, plain, rtol=1e-12, atol=1e-12)
    again = pk.a_orthogonalize_against(A, plain, Q)
    assert np.linalg.norm(again - plain) <= 1e-12 * np.linalg.norm(plain)
    # against the oracle's CGS2 (cached A Q, the engine's form)
    ref = orc.cgs2_project(W.copy(), [(Q, D @ Q)])
    np.testing.assert_allclose(cached, ref, rtol=1e-11, atol=1e-12)


def test_orthogonalize_shape_errors(rng):
    with pytest.raises(ValueError):
        pk.a_orthogonalize_against(eye_csr(5), rng.standard_normal((5, 2)), rng.standard_normal((4, 2)))


def test_a_cholqr_invariants(rng):
    A = eye_csr(8)
    Q, _ = np.linalg.qr(rng.standard_normal((8, 3)))
    np.testing.assert_allclose(pk.a_cholqr(A, Q), Q, rtol=1e-13, atol=1e-13)        # fixed point
    np.testing.assert_allclose(pk.a_cholqr(A, 3.0 * Q), Q, rtol=1e-12, atol=1e-12)  # scale removed
    B, D = spd_csr(13, rng)
    assert a_err(pk.a_cholqr(B, rng.standard_normal((13, 4))), D) <= 1e-10
    w = rng.standard_normal((8, 1))
    with pytest.raises(pk.Breakdown):
        pk.a_cholqr(A, np.hstack([w, w]))


def test_pre_cholqr_invariants_and_oracle(rng):
    A, D = spd_csr(10, rng)
    W = rng.standard_normal((10, 3))
    assert np.max(np.abs(pk.pre_cholqr(eye_csr(10), W).T @ pk.pre_cholqr(eye_csr(10), W) - np.eye(3))) <= 1e-12
    out = pk.pre_cholqr(A, W)
    assert a_err(out, D) <= 1e-10
    # the oracle's Pre-CholQR (normalize_block, aortho.py:98-110) returns the same block
    ref, _ = orc.pre_cholqr_block(W.copy(), lambda X: D @ X)
    np.testing.assert_allclose(out, ref, rtol=1e-11, atol=1e-12)
    # spans are preserved: each output column lies in span(W)
    P = W @ np.linalg.pinv(W)
    assert np.max(np.abs(P @ out - out)) <= 1e-8 * np.max(np.abs(out))
    with pytest.raises(pk.Breakdown, match="zero column 1 entering Pre-CholQR"):
        pk.pre_cholqr(A, np.column_stack([W[:, 0], np.zeros(10), W[:, 2]]))


def test_pre_cholqr_tames_ill_scaled_columns(rng):
    A, D = spd_csr(16, rng, lo=1.0, hi=100.0)
    W = rng.standard_normal((16, 3)) * np.array([1e4, 1.0, 1e-4])
    pre_err = a_err(pk.pre_cholqr(A, W), D)
    assert pre_err <= 1e-10
    try:
        plain_err = a_err(pk.a_cholqr(A, W), D)
    except pk.Breakdown:
        return
    assert plain_err >= 100.0 * max(pre_err, 1e-16)


def test_project_then_normalize_keeps_basis_orthonormal(rng):
    A, D = spd_csr(30, rng, lo=1.0, hi=1e4)
    Q = pk.pre_cholqr(A, rng.standard_normal((30, 3)))
    W = pk.pre_cholqr(A, pk.a_orthogonalize_against(A, rng.standard_normal((30, 3)), Q))
    assert a_err(np.hstack([Q, W]), D) <= 1e-10


def test_torch_in_torch_out(rng):
    A, D = spd_csr(9, rng)
    W = torch.from_numpy(rng.standard_normal((9, 2))).cuda()
    out = pk.pre_cholqr(A, W)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    assert a_err(out.cpu().numpy(), D) <= 1e-10


@pytest.mark.parametrize("cond", [1e2, 1e4, 1e6])
@pytest.mark.parametrize("m", [16, 64])
def test_pre_cholqr_ill_conditioned_matches_substitution(rng, cond, m):
    """The device applies R^-1 as an explicit upper inverse (DMMA block product) where the
    reference substitutes (solve_triangular, linalg.py:187-196).  Across Pre-CholQR's operating
    range (kappa(W) up to ~1e7: the Cholesky of W^T W sees kappa^2; beyond it both break down,
    test_pre_cholqr_breakdown_matches_reference) the device result is as A-orthonormal as the
    reference algorithm's (the oracle) and spans the same space."""
    n = 3000
    A, D = spd_csr(n, rng, 1.0, 100.0)
    U, _ = np.linalg.qr(rng.standard_normal((n, m)))
    V, _ = np.linalg.qr(rng.standard_normal((m, m)))
    W = (U * np.geomspace(1.0, 1.0 / cond, m)) @ V.T
    ours = pk.pre_cholqr(A, W)
    ref, _ = orc.pre_cholqr_block(W.copy(), lambda X: D @ X)
    e_ours, e_ref = a_err(ours, D), a_err(ref, D)
    assert e_ours <= 10.0 * e_ref + 1e-12, (e_ours, e_ref)
    # same column space: the projection of ours onto the reference basis loses nothing
    G = ref.T @ D @ ours
    assert np.linalg.norm(ref @ G - ours) <= 1e-6 * np.linalg.norm(ours), np.linalg.norm(ref @ G - ours)


@pytest.mark.parametrize("m", [16, 64])
def test_pre_cholqr_breakdown_matches_reference(rng, m):
    """kappa(W) = 1e10: the Gram W^T W is singular to working precision; the device and the
    reference algorithm both raise Breakdown (linalg.py:178-183) rather than return a basis."""
    n = 3000
    A, D = spd_csr(n, rng, 1.0, 100.0)
    U, _ = np.linalg.qr(rng.standard_normal((n, m)))
    V, _ = np.linalg.qr(rng.standard_normal((m, m)))
    W = (U * np.geomspace(1.0, 1e-10, m)) @ V.T  # mixed columns: unit scaling cannot undo it
    with pytest.raises(pk.Breakdown):
        pk.pre_cholqr(A, W)
    with pytest.raises(orc.OracleBreakdown):
        orc.pre_cholqr_block(W.copy(), lambda X: D @ X)
