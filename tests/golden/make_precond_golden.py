"""Golden preconditioned solves from the real reference (blockjacobi.py, solvers.py:282-316).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_precond_golden.py

Writes tests/golden/precond.npz + precond.json (inputs and reports).
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, os.environ.get("EKCG_REFERENCE", "/root/reference/pkg/src"))
import ekcg  # noqa: E402

OUT = Path(__file__).resolve().parent


def random_spd(n, rng):
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    D = (Q * (1.0 + 9.0 * rng.random(n))) @ Q.T
    return 0.5 * (D + D.T)


def main():
    cases = []
    A = ekcg.gen_poisson2d(12, 12)
    b, xs = ekcg.make_rhs(A, 16)
    for method in ("sre-cg2", "sre-cg", "msdo-cg", "modified-msdo-cg"):
        for mode in ("modified", "explicit-hat"):
            cases.append((f"p12_{method}_{mode}", A, b, xs, None, 4, 4, "chol", dict(method=method, t=4, precond_mode=mode)))
    A8 = ekcg.gen_poisson2d(8, 8)
    b8, _ = ekcg.make_rhs(A8, 18)
    for mode in ("modified", "explicit-hat"):
        cases.append((f"p8_misaligned_{mode}", A8, b8, None, None, 3, 4, "chol", dict(method="sre-cg2", t=3, precond_mode=mode)))
    A10 = ekcg.gen_poisson2d(10, 10)
    b10, _ = ekcg.make_rhs(A10, 41)
    x0 = np.random.default_rng(12345).standard_normal(A10.n)
    for mode in ("modified", "explicit-hat"):
        cases.append((f"p10_x0_{mode}", A10, b10, None, x0, 4, 4, "chol", dict(method="sre-cg2", t=4, precond_mode=mode)))
    As = ekcg.gen_skyscraper(12, 12, contrast=1e4)
    bs, _ = ekcg.make_rhs(As, 5)
    cases.append(("sky12_ichol0", As, bs, None, None, 4, 4, "ichol0", dict(method="sre-cg2", t=4)))
    rng = np.random.default_rng(12345)
    D = random_spd(12, rng)
    rows, cols = np.nonzero(D)
    Ar = ekcg.SparseSpdMatrix.from_coo(12, rows, cols, D[rows, cols])
    br = rng.standard_normal(12)
    cases.append(("rand12_exact", Ar, br, None, None, 2, 1, "chol", dict(method="sre-cg2", t=2)))
    A16 = ekcg.gen_poisson2d(16, 16)
    b16, _ = ekcg.make_rhs(A16, 19)
    cases.append(("p16_msdo_switch", A16, b16, None, None, 4, 4, "chol", dict(method="msdo-cg", t=4, switch_tol=1e-5)))

    meta, arrays = {}, {}
    for name, A, b, xs, x0, t, nblocks, kind, kw in cases:
        F = ekcg.build_block_jacobi(A, ekcg.uniform_block_bounds(A.n, nblocks), kind=kind)
        p = ekcg.contiguous_partition(A.n, t)
        _, rep = ekcg.enlarged_solve(A, b, x0=x0, partition=p, x_star=xs,
                                     cfg=ekcg.SolverConfig(preconditioner=F, **kw))
        meta[name] = {"cfg": kw, "nblocks": nblocks, "kind": kind, "status": rep.status,
                      "iterations": int(rep.iterations), "notes": list(rep.notes),
                      "peak_block_vectors": int(rep.peak_block_vectors), "switch_iteration": rep.switch_iteration,
                      "true_residual": float(rep.true_residual),
                      "relative_error": None if rep.relative_error is None else float(rep.relative_error)}
        arrays[f"{name}__history"] = rep.residual_history
        arrays[f"{name}__x"] = rep.x
        arrays[f"{name}__rp"], arrays[f"{name}__ci"], arrays[f"{name}__vals"] = A.row_ptr, A.col_idx, A.values
        arrays[f"{name}__b"] = b
        if x0 is not None:
            arrays[f"{name}__x0"] = x0
        if xs is not None:
            arrays[f"{name}__xs"] = xs
        for i, L in enumerate(F.factors):
            arrays[f"{name}__L{i}"] = L
        print(name, rep.status, rep.iterations, rep.notes)
    (OUT / "precond.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    np.savez_compressed(OUT / "precond.npz", **arrays)


if __name__ == "__main__":
    main()
