"""The package's input generators reproduce the reference generators bit for bit."""

import hashlib

import numpy as np
import pytest

import paper_2305_19013_b200 as pk
from paper_2305_19013_b200.problems import make_config


def csr_hash(A):
    h = hashlib.sha256()
    for arr in (A.row_ptr.astype(np.int64), A.col_idx.astype(np.int64), A.values.astype(np.float64)):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


GENS = {
    "poisson2d_100": lambda: pk.gen_poisson2d(100, 100),
    "poisson3d_16": lambda: pk.gen_poisson3d(16, 16, 16),
    "poisson3d_64": lambda: pk.gen_poisson3d(64, 64, 64),
    "skyscraper2d_12_1e4": lambda: pk.gen_skyscraper(12, 12, contrast=1e4),
    "skyscraper3d_10_11_12": lambda: pk.gen_skyscraper(10, 11, 12),
    "aniso3d_6_100": lambda: pk.gen_aniso3d(6, 6, 6, 100.0),
    "cfg3_16": lambda: make_config(3, 16, device_rhs=False).csr(),
    "cfg3_32": lambda: make_config(3, 32, device_rhs=False).csr(),
    "cfg5_64": lambda: make_config(5, 64, device_rhs=False).csr(),
    "cfg5_256": lambda: make_config(5, 256, device_rhs=False).csr(),
}


@pytest.mark.parametrize("name", sorted(GENS))
def test_generator_bitwise(generators_golden, name):
    A = GENS[name]()
    ref = generators_golden[name]
    assert (A.n, A.nnz) == (ref["n"], ref["nnz"])
    assert csr_hash(A) == ref["sha256"]


@pytest.mark.parametrize("idx,edge", [(1, 100), (2, 16), (2, 64), (3, 16), (3, 32), (5, 64), (5, 256)])
def test_config_rhs_and_partition(generators_golden, idx, edge):
    prob = make_config(idx, edge, device_rhs=False)
    ref = generators_golden[f"cfg{idx}_{edge}_rhs"]
    assert hashlib.sha256(np.ascontiguousarray(prob.b).tobytes()).hexdigest() == ref["b_sha256"]
    owner = prob.partition.owner().astype(np.int64)
    assert hashlib.sha256(owner.tobytes()).hexdigest() == ref["owner_sha256"]


def test_validated_matrix_roundtrip():
    A = pk.gen_poisson3d(5, 4, 3)
    B = pk.SparseSpdMatrix(A.n, A.row_ptr, A.col_idx, A.values)  # validates
    assert B.nnz == A.nnz
    D = A.to_dense()
    C = pk.SparseSpdMatrix.from_coo(A.n, *np.nonzero(D), D[np.nonzero(D)])
    assert np.array_equal(C.values, A.values)


def test_matrix_validation_errors():
    with pytest.raises(ValueError, match="symmetric"):
        pk.SparseSpdMatrix.from_coo(2, [0, 0, 1], [0, 1, 1], [2.0, 1.0, 2.0])
    with pytest.raises(ValueError, match="diagonal"):
        pk.SparseSpdMatrix.from_coo(2, [0, 1, 1], [1, 0, 1], [1.0, 1.0, 2.0])


def test_box_owner_layout():
    owner = pk.problems.box_owner((8, 4, 4), (4, 2, 2))
    grid = owner.reshape(4, 4, 8)  # (z, y, x)
    assert grid[0, 0, 0] == 0 and grid[0, 0, 7] == 3 and grid[0, 3, 0] == 4 and grid[3, 0, 0] == 8
    assert np.array_equal(np.bincount(owner), np.full(16, 8))


def test_stencil_descriptor_host_csr():
    prob = make_config(5, 64, device_rhs=False)
    from paper_2305_19013_b200.problems import diffusion_csr
    A = diffusion_csr(prob.shape, prob.node_kappa())
    assert csr_hash(A) == csr_hash(prob.csr())


def test_from_coo_sums_duplicates_and_validates():
    """from_coo (linalg.py:55-79): duplicates summed, CSR rows sorted; the validator's
    messages for each malformed input (linalg.py:81-109)."""
    rng = np.random.default_rng(4)
    for _ in range(50):
        n = int(rng.integers(1, 20))
        k = int(rng.integers(0, 60))
        r, c, v = rng.integers(0, n, k), rng.integers(0, n, k), rng.standard_normal(k)
        keep = r != c  # off-diagonal pairs (duplicates summed in the same order on both sides)
        r, c, v = np.minimum(r, c)[keep], np.maximum(r, c)[keep], v[keep]
        R = np.concatenate([r, c, np.arange(n), np.arange(n)])
        C = np.concatenate([c, r, np.arange(n), np.arange(n)])
        V = np.concatenate([v, v, np.full(n, 40.0), np.full(n, 0.5)])
        A = pk.SparseSpdMatrix.from_coo(n, R, C, V)
        D = np.zeros((n, n))
        np.add.at(D, (R, C), V)
        assert np.allclose(A.to_dense(), D, rtol=1e-15, atol=0)
        assert np.array_equal(A.diagonal(), np.diag(A.to_dense()))
        assert all(np.all(np.diff(A.col_idx[A.row_ptr[i]:A.row_ptr[i + 1]]) > 0) for i in range(n))
    bad = [((2, [0, 2, 1], [0, 1], [1.0, 1.0]), "malformed row_ptr"),
           ((2, [0, 2, 2], [1, 0], [1.0, 1.0]), "sorted and unique"),
           ((2, [0, 1, 2], [0, 0], [1.0, 1.0]), "diagonal entries"),
           ((2, [0, 1, 2], [0, 1], [1.0, -1.0]), "diagonal entries"),
           ((2, [0, 2, 3], [0, 1, 1], [2.0, 1.0, 2.0]), "symmetric"),
           ((2, [0, 1, 2], [0, 1], [np.inf, 1.0]), "finite"),
           ((2, [0, 1, 2], [0, 5], [1.0, 1.0]), "out of range")]
    for args, msg in bad:
        with pytest.raises(ValueError, match=msg):
            pk.SparseSpdMatrix(*args)
    with pytest.raises(ValueError, match="out of range"):
        pk.SparseSpdMatrix.from_coo(3, [0, 3], [0, 0], [1.0, 1.0])
