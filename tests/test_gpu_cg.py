"""Classical CG on the device (the `cg` that enlarged_solve dispatches to,
solvers.py:199-258, 271-272) against runs of the real reference
(tests/golden/cg.json, made by tests/golden/make_cg_golden.py)."""

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2305_19013_b200 as pk
from paper_2305_19013_b200.reporting import run_batch

GOLDEN = json.loads((Path(__file__).resolve().parent / "golden" / "cg.json").read_text())


def build(recipe):
    g = recipe["gen"]
    A = pk.gen_poisson2d(*g[1:]) if g[0] == "poisson2d" else pk.gen_poisson3d(*g[1:])
    kind, _, seed = recipe["xstar"].partition(":")
    if kind == "normal":
        x_star = np.random.default_rng(int(seed)).standard_normal(A.n)
        b = pk.spmv(A, x_star)
    else:
        b, x_star = pk.make_rhs(A, int(seed))
    x0 = None
    if "x0" in recipe:
        x0 = np.random.default_rng(int(recipe["x0"].split(":")[1])).standard_normal(A.n)
    F = None
    if "precond" in recipe:
        kind_, nb = recipe["precond"]
        F = pk.build_block_jacobi(A, pk.uniform_block_bounds(A.n, nb), kind=kind_)
    return A, b, x_star, x0, F


@pytest.mark.parametrize("name", sorted(GOLDEN["cases"]))
@pytest.mark.parametrize("entry", ["cg", "enlarged_solve"])
def test_cg_matches_reference(name, entry):
    ref = GOLDEN["cases"][name]
    A, b, x_star, x0, F = build(ref["recipe"])
    cfg = pk.SolverConfig(method="cg", preconditioner=F, **ref["recipe"]["kw"])
    if entry == "cg":
        x, rep = pk.cg(A, b, x0=x0, cfg=cfg, x_star=x_star)
    else:
        x, rep = pk.enlarged_solve(A, b, x0=x0, cfg=cfg, x_star=x_star)
    assert isinstance(x, np.ndarray) and x.shape == (A.n,)
    assert rep.status == ref["status"]
    assert abs(rep.iterations - ref["iterations"]) <= max(1, round(0.02 * ref["iterations"]))
    h, g = np.asarray(rep.residual_history), np.asarray(ref["history"])
    n = min(len(h), len(g), 21)
    assert np.max(np.abs(h[:n] / h[0] - g[:n] / g[0]) / (g[:n] / g[0])) <= 1e-8
    assert rep.peak_block_vectors == 0 and rep.notes == ref["notes"]
    assert rep.true_residual <= max(2 * ref["true_residual"], 1e-8 * np.linalg.norm(b))
    assert abs(rep.relative_error - ref["relative_error"]) <= 1e-6 * max(1.0, ref["relative_error"])


def test_cg_zero_rhs_and_validation():
    A = pk.gen_poisson2d(6, 6)
    x, rep = pk.cg(A, np.zeros(A.n))
    assert rep.status == "converged" and rep.iterations == 0 and not np.any(x)
    with pytest.raises(ValueError):
        pk.cg(A, np.zeros(A.n), cfg=pk.SolverConfig(method="sre-cg2", t=2))
    with pytest.raises(ValueError):
        pk.cg(A, np.zeros(A.n + 1))


def _rows(text):
    lines = text.strip().splitlines()
    hdr = lines[0].split(",")
    return [dict(zip(hdr, l.split(","))) for l in lines[1:]]


def test_preconditioned_batch_matches_reference(tmp_path):
    """runs.csv / history TSVs of a bj-chol batch (cg + SRE-CG2 cells) against the
    reference's own run_experiment output."""
    gold = GOLDEN["batch"]
    run_batch(gold["spec"], tmp_path)
    ours, ref = _rows((tmp_path / "runs.csv").read_text()), _rows(gold["csv"])
    assert [r["run_id"] for r in ours] == [r["run_id"] for r in ref]
    for a, b in zip(ours, ref):
        for col in ("matrix", "method", "t", "partition", "retention", "precond", "precond_blocks",
                    "precond_mode", "status", "peak_block_vectors"):
            assert a[col] == b[col], (a["run_id"], col, a[col], b[col])
        assert abs(int(a["iterations"]) - int(b["iterations"])) <= 1
        ha = np.array([float(l.split("\t")[1]) for l in (tmp_path / f"{a['run_id']}_history.tsv").read_text()
                       .strip().splitlines()[1:]])
        hb = np.array([float(l.split("\t")[1]) for l in gold["histories"][f"{b['run_id']}_history.tsv"]
                       .strip().splitlines()[1:]])
        n = min(len(ha), len(hb), 21)
        keep = hb[:n] / hb[0] > 1e-6  # preconditioned runs reach round-off within ~15 iterations
        assert np.max(np.abs(ha[:n][keep] / ha[0] - hb[:n][keep] / hb[0]) / (hb[:n][keep] / hb[0])) <= 1e-8


def test_cg_breakdown_on_nonpositive_curvature():
    """An indefinite matrix (positive diagonal) stops CG with the reference's status and note."""
    ref = GOLDEN["indefinite"]
    d = ref["input"]
    A = pk.SparseSpdMatrix.from_coo(d["n"], np.array(d["rows"]), np.array(d["cols"]), np.array(d["vals"]))
    _, rep = pk.cg(A, np.array(d["b"]))
    assert rep.status == ref["status"] == "breakdown"
    assert rep.iterations == ref["iterations"]
    assert rep.notes == ref["notes"]
    np.testing.assert_allclose(rep.residual_history, ref["history"], rtol=1e-12)
