"""Golden classical-CG runs of the real reference (`ekcg.cg`, solvers.py:199-258).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cg_golden.py

Writes tests/golden/cg.json: for each case the inputs' recipe, the residual
history, status, iteration count, true residual and relative error; plus a
preconditioned batch (`bj-chol` / `bj-ichol0`, cg and an enlarged method) of
`ekcg.run_experiment` as runs.csv + history TSVs.
"""
import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, os.environ.get("EKCG_REFERENCE", "/root/reference/pkg/src"))
import ekcg  # noqa: E402
from ekcg.harness import run_experiment  # noqa: E402

CASES = {
    # BASELINE config 1's operator and right-hand side (x* ~ N(0,1) seed 0), classical CG
    "cfg1_cg": {"gen": ["poisson2d", 100, 100], "xstar": "normal:0", "kw": {}},
    # block-Jacobi (dense Cholesky blocks) preconditioned CG
    "p12_pcg_bjchol4": {"gen": ["poisson2d", 12, 12], "xstar": "rhs:312", "kw": {}, "precond": ["chol", 4]},
    # incomplete-Cholesky blocks, from a nonzero x0, capped iterations
    "p3d8_pcg_ichol0_kmax": {"gen": ["poisson3d", 8, 8, 8], "xstar": "rhs:5", "kw": {"kmax": 6},
                             "precond": ["ichol0", 4], "x0": "normal:9"},
}
# an indefinite matrix with a positive diagonal: CG stops on nonpositive curvature
INDEFINITE = {"n": 3, "rows": [0, 0, 1, 1, 2, 1, 2], "cols": [0, 1, 0, 1, 2, 2, 1],
              "vals": [1.0, 2.0, 2.0, 1.0, 1.0, 0.5, 0.5], "b": [1.0, 0.0, 1.0]}
BATCH = {"matrix": "poisson2d:10,10", "methods": ["cg", "sre-cg2"], "t": [2], "retention": ["full"],
         "precond": "bj-chol:4", "precond_mode": "modified", "tol": 1e-8, "seed": 7}


def build(case):
    g = case["gen"]
    A = ekcg.gen_poisson2d(*g[1:]) if g[0] == "poisson2d" else ekcg.gen_poisson3d(*g[1:])
    kind, _, seed = case["xstar"].partition(":")
    if kind == "normal":
        x_star = np.random.default_rng(int(seed)).standard_normal(A.n)
        b = ekcg.spmv(A, x_star)
    else:
        b, x_star = ekcg.make_rhs(A, int(seed))
    x0 = None
    if "x0" in case:
        x0 = np.random.default_rng(int(case["x0"].split(":")[1])).standard_normal(A.n)
    F = None
    if "precond" in case:
        kind_, nb = case["precond"]
        F = ekcg.build_block_jacobi(A, ekcg.uniform_block_bounds(A.n, nb), kind=kind_)
    return A, b, x_star, x0, F


if __name__ == "__main__":
    out = {"cases": {}}
    for name, case in CASES.items():
        A, b, x_star, x0, F = build(case)
        cfg = ekcg.SolverConfig(method="cg", preconditioner=F, **case["kw"])
        x, rep = ekcg.cg(A, b, x0=x0, cfg=cfg, x_star=x_star)
        out["cases"][name] = {"recipe": case, "status": rep.status, "iterations": rep.iterations,
                              "history": [float(v) for v in rep.residual_history],
                              "true_residual": rep.true_residual, "relative_error": rep.relative_error,
                              "notes": rep.notes}
    d = INDEFINITE
    A = ekcg.SparseSpdMatrix.from_coo(d["n"], np.array(d["rows"]), np.array(d["cols"]), np.array(d["vals"]))
    _, rep = ekcg.cg(A, np.array(d["b"]))
    out["indefinite"] = {"input": d, "status": rep.status, "iterations": rep.iterations, "notes": rep.notes,
                         "history": [float(v) for v in rep.residual_history]}
    with tempfile.TemporaryDirectory() as tmp:
        run_experiment(BATCH, tmp, render_figures=False)
        out["batch"] = {"spec": BATCH, "csv": (Path(tmp) / "runs.csv").read_text(),
                        "histories": {p.name: p.read_text() for p in sorted(Path(tmp).glob("*_history.tsv"))}}
    (Path(__file__).resolve().parent / "cg.json").write_text(json.dumps(out, indent=1))
    print({k: (v["status"], v["iterations"]) for k, v in out["cases"].items()})
