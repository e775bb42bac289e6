"""Pin the CPU oracle (oracle/ekcg_oracle.py) to the REAL reference's outputs.

The golden fixtures were produced by running `ekcg` itself
(tests/golden/make_golden.py).  The oracle uses the same numpy/BLAS
primitives in the same order, so on the same host its results are bitwise
those of the reference; the assertions below demand exactly that wherever the
computation is host-deterministic.
"""

import numpy as np
import pytest

from conftest import golden_case_inputs
from oracle import ekcg_oracle as orc


def test_split_known_answer(kernels_golden):
    g = kernels_golden
    W = orc.split_block(g["split_owner"], 3, g["split_v"])
    assert np.array_equal(W, g["split_W"])
    assert np.array_equal(W.sum(axis=1), g["split_v"])  # one copied entry per row


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_spmm_spmv_bitwise(kernels_golden, tag):
    g = kernels_golden
    rp, ci, v, X = g[f"spmm_{tag}_rp"], g[f"spmm_{tag}_ci"], g[f"spmm_{tag}_v"], g[f"spmm_{tag}_X"]
    assert np.array_equal(orc.csr_spmm(rp, ci, v, X), g[f"spmm_{tag}_Y"])
    assert np.array_equal(orc.csr_spmv(rp, ci, v, X[:, 3].copy()), g[f"spmv_{tag}_y"])


@pytest.mark.parametrize("tag", ["a", "c"])
def test_pairwise_association_model(kernels_golden, tag):
    """y_i = p_0 + pairwise(p_1..p_k): the association the CUDA kernels implement."""
    g = kernels_golden
    rp, ci, v, X, Y = (g[f"spmm_{tag}_{k}"] for k in ("rp", "ci", "v", "X", "Y"))
    for col in (0, 5, 69):
        for i in range(len(rp) - 1):
            lo, hi = rp[i], rp[i + 1]
            p = [v[j] * X[ci[j], col] for j in range(lo, hi)]
            y = p[0] + orc.pairwise_tail(p[1:]) if len(p) > 1 else p[0]
            assert y == Y[i, col]


def test_small_dense_kernels(kernels_golden):
    g = kernels_golden
    assert np.array_equal(orc.small_cholesky(g["chol_2x2_B"]), np.array([[2.0, 1.0], [0.0, 2.0]]))
    assert np.array_equal(orc.small_cholesky(g["chol_rand_B"]), g["chol_rand_R"])
    assert np.array_equal(orc.right_tri_solve(g["trsm_X"], g["trsm_R"]), g["trsm_Y"])
    assert np.allclose(g["gram_X"].T @ g["gram_Y"], g["gram_G"], rtol=1e-14, atol=0)
    with pytest.raises(orc.OracleBreakdown, match="pivot"):
        orc.small_cholesky(np.array([[1.0, 1.0], [1.0, 1.0]]))


def _run_small(meta, arrays, name, **over):
    rp, ci, vals, b, owner, x0 = golden_case_inputs(arrays, name)
    kw = dict(meta[name]["cfg"])
    kw.update(over)
    t = kw.pop("t")
    return orc.run_oracle(rp, ci, vals, b, owner, t, x0=x0, **kw)


SMALL = [
    "p12_srecg2_t4_full", "p12_srecg2_t4_trunc3", "p12_srecg2_t8_trunc2", "p12_msdo_t4",
    "p12_modmsdo_t4", "p12_srecg2_t16_full", "p12_srecg2_t32_trunc4", "p10_srecg_t2",
    "p10_srecg2_t2_trunc2", "p10_maxiter_t2", "p10_t1", "p10_x0_t4", "p12_restart5_t2",
    "sky12_restarttol_t2", "sky20_stagnation_t2", "p16_switch_t4", "p16_switch_trunc4_t4",
    "p20_trueres25_t2", "p4_breakdown_t2", "identity12_t4", "p8_zero_rhs_t2", "aniso6_box222_t8",
]


@pytest.mark.parametrize("name", SMALL)
def test_oracle_matches_reference_solve(solves_golden, name):
    meta, arrays = solves_golden
    ref = meta[name]
    out = _run_small(meta, arrays, name)
    assert out["status"] == ref["status"]
    assert out["iterations"] == ref["iterations"]
    assert np.array_equal(out["residual_history"], arrays[f"{name}__history"])
    assert np.array_equal(out["x"], arrays[f"{name}__x"])
    assert out["peak_block_vectors"] == ref["peak_block_vectors"]
    assert out["restart_iterations"] == ref["restart_iterations"]
    assert out["switch_iteration"] == ref["switch_iteration"]
    assert out["notes"] == ref["notes"]
    assert [[k, v] for k, v in out["true_residual_checks"]] == ref["true_residual_checks"]
    assert out["true_residual"] == ref["true_residual"]


@pytest.mark.parametrize("name,edge,kmax", [("cfg1_100", 100, None), ("cfg2_16", 16, None),
                                            ("cfg3_16", 16, 25), ("cfg5_64", 64, 25)])
def test_oracle_matches_reference_configs(solves_golden, name, edge, kmax):
    """Config inputs from the package generator (pinned in test_problems) through the oracle."""
    from paper_2305_19013_b200.problems import make_config
    meta, arrays = solves_golden
    idx = int(name[3])
    prob = make_config(idx, edge, device_rhs=False)
    A = prob.csr()
    kw = dict(prob.solver_kwargs)
    t = kw.pop("t")
    if kmax is not None:
        kw["kmax"] = kmax
    out = orc.run_oracle(A.row_ptr, A.col_idx, A.values, prob.b, prob.partition.owner(), t,
                         x_star=prob.x_star, **kw)
    hist = arrays[f"{name}__history"]
    if kmax is None:
        assert out["iterations"] == meta[name]["iterations"]
        assert out["status"] == meta[name]["status"]
        assert np.array_equal(out["residual_history"], hist)
        assert out["true_residual"] == meta[name]["true_residual"]
    else:
        assert np.array_equal(out["residual_history"], hist[: kmax + 1])


def test_sstep_s1_is_srecg2(solves_golden):
    meta, arrays = solves_golden
    a = _run_small(meta, arrays, "p12_srecg2_t4_trunc3", s=1)
    assert np.array_equal(a["residual_history"], arrays["p12_srecg2_t4_trunc3__history"])


def test_sstep_converges_in_fewer_outer_iterations(solves_golden):
    """s-step (unpinned beyond s=1): s=2 on the same system needs about half the iterations."""
    meta, arrays = solves_golden
    one = _run_small(meta, arrays, "p12_srecg2_t4_full")
    two = _run_small(meta, arrays, "p12_srecg2_t4_full", s=2)
    assert two["status"] == "converged"
    assert two["iterations"] <= (one["iterations"] + 1) // 2 + 2
    assert two["peak_block_vectors"] == 8 * two["iterations"]


@pytest.mark.parametrize("idx,edge,kmax", [(4, 16, 5), (5, 64, 10), (3, 16, 8), (2, 12, 200)])
def test_lowmem_oracle_matches(idx, edge, kmax):
    """The bounded-memory restatement used for the full-size fixtures (row-chunked
    products, A Q recomputed) is bitwise run_oracle, here with 37-row chunks."""
    from paper_2305_19013_b200.problems import make_config
    prob = make_config(idx, edge, device_rhs=False)
    A = prob.csr()
    kw = dict(prob.solver_kwargs, kmax=kmax)
    t = kw.pop("t")
    ref = orc.run_oracle(A.row_ptr, A.col_idx, A.values, prob.b, prob.partition.owner(), t, **kw)
    low = orc.run_oracle_lowmem(A.row_ptr, A.col_idx, A.values, prob.b, prob.partition.owner(), t,
                                chunk_rows=37, **kw)
    assert low["status"] == ref["status"] and low["iterations"] == ref["iterations"]
    assert np.array_equal(low["residual_history"], ref["residual_history"])
    assert np.array_equal(low["x"], ref["x"])
    assert low["peak_block_vectors"] == ref["peak_block_vectors"]


def test_chunked_spmm_bitwise(kernels_golden):
    g = kernels_golden
    for tag in ("a", "b", "c"):
        rp, ci, v, X = g[f"spmm_{tag}_rp"], g[f"spmm_{tag}_ci"], g[f"spmm_{tag}_v"], g[f"spmm_{tag}_X"]
        assert np.array_equal(orc.csr_spmm_chunked(rp, ci, v, X, 7), g[f"spmm_{tag}_Y"])
        assert np.array_equal(orc.csr_spmm_chunked(rp, ci, v, X[:, 3].copy(), 11), g[f"spmv_{tag}_y"])


def test_full_size_fixture_inputs():
    """The full-size fixtures (make_full_golden.py) were built from the same inputs the
    package's generators produce: b, owner map, and (cfg3) the reference generator's CSR."""
    import hashlib
    import json
    from pathlib import Path
    from paper_2305_19013_b200.problems import make_config
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    gold = Path(__file__).resolve().parent / "golden"
    p3 = gold / "full_cfg3.json"
    if p3.exists():
        fx = json.loads(p3.read_text())
        prob = make_config(3, fx["edge"], device_rhs=False)
        assert sha(prob.b) == fx["b_sha256"] and sha(prob.partition.owner()) == fx["owner_sha256"]
        A = prob.csr()
        h = hashlib.sha256()
        for arr in (A.row_ptr.astype(np.int64), A.col_idx.astype(np.int64), A.values.astype(np.float64)):
            h.update(np.ascontiguousarray(arr).tobytes())
        assert h.hexdigest() == fx["csr_sha256"]
    p5 = gold / "full_cfg5.json"
    if p5.exists():
        fx = json.loads(p5.read_text())
        prob = make_config(5, fx["edge"], device_rhs=False)
        assert sha(prob.b) == fx["b_sha256"] and sha(prob.partition.owner()) == fx["owner_sha256"]
        assert sha(prob.kappa_field) == fx["kappa_field_sha256"]
