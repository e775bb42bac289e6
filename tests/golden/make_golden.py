"""Generate the golden fixtures by running the REAL reference (`ekcg`).

Run in the build container only (the reference is importable there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--skip-cfg2]

Writes tests/golden/{kernels.npz, generators.json, solves.json, solves.npz}.
The GPU box never reads /root/reference: tests consume only these files.
Inputs are built with the reference's own generators; the package's
generators are pinned to them through generators.json.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = os.environ.get("EKCG_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)
import ekcg  # noqa: E402
from ekcg.generators import _diffusion_matrix  # noqa: E402

OUT = Path(__file__).resolve().parent
ROOT = OUT.parent.parent
sys.path.insert(0, str(ROOT))


def csr_hash(A):
    h = hashlib.sha256()
    for arr in (A.row_ptr.astype(np.int64), A.col_idx.astype(np.int64), A.values.astype(np.float64)):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


def arr_hash(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------------------
# input builders (reference side; the package's make_config must agree)
# ---------------------------------------------------------------------------

def box_subdomains(shape, boxes):
    ids = [(np.arange(s) * b) // s for s, b in zip(shape, boxes)]
    grid = np.zeros(shape[::-1], dtype=np.int64)
    mult = 1
    for ax, (bid, b) in enumerate(zip(ids, boxes)):
        sh = [1] * len(shape)
        sh[len(shape) - 1 - ax] = bid.size
        grid = grid + mult * bid.reshape(sh)
        mult *= b
    owner = grid.reshape(-1)
    t = int(np.prod(boxes))
    return owner, ekcg.Partition(owner.size, [np.flatnonzero(owner == j) for j in range(t)])


def config_inputs(index, N):
    """(A, b, x_star, partition, cfg kwargs) for BASELINE config `index` at edge N."""
    if index == 1:
        A = ekcg.gen_poisson2d(N, N)
        x_star = np.random.default_rng(0).standard_normal(A.n)
        return A, ekcg.spmv(A, x_star), x_star, ekcg.contiguous_partition(A.n, 8), dict(method="sre-cg", t=8)
    if index == 2:
        A = ekcg.gen_poisson3d(N, N, N)
        x_star = np.random.default_rng(1).standard_normal(A.n)
        _, p = box_subdomains((N, N, N), (4, 2, 2))
        return A, ekcg.spmv(A, x_star), x_star, p, dict(method="sre-cg2", t=16)
    if index == 3:
        cell = N // 8
        i = np.arange(N) // cell
        kap = np.where(((i[None, None, :] % 2) == 0) & ((i[None, :, None] % 2) == 0), 1000.0, 1.0)
        kap = np.broadcast_to(kap, (N, N, N)).reshape(-1)
        A = _diffusion_matrix((N, N, N), kap)
        b = np.random.default_rng(2).uniform(-1.0, 1.0, A.n)
        _, p = box_subdomains((N, N, N), (4, 4, 2))
        return A, b, None, p, dict(method="sre-cg2", t=32, retention="trunc", trunc=4)
    if index == 5:
        nt = N // 16
        field = np.exp(np.random.default_rng(4).uniform(np.log(1e-3), np.log(1e3), (nt, nt)))
        kap = np.repeat(np.repeat(field, 16, axis=0), 16, axis=1).reshape(-1)
        A = _diffusion_matrix((N, N), kap)
        b = np.random.default_rng(5).uniform(-1.0, 1.0, A.n)
        _, p = box_subdomains((N, N), (8, 8))
        return A, b, None, p, dict(method="sre-cg2", t=64, retention="trunc", trunc=3, tol=1e-6)
    raise ValueError(index)


def report_dict(rep, keep_x):
    d = {
        "status": rep.status,
        "iterations": int(rep.iterations),
        "switch_iteration": rep.switch_iteration,
        "restart_iterations": [int(k) for k in rep.restart_iterations],
        "peak_block_vectors": int(rep.peak_block_vectors),
        "true_residual": float(rep.true_residual),
        "relative_error": None if rep.relative_error is None else float(rep.relative_error),
        "true_residual_checks": [[int(k), float(v)] for k, v in rep.true_residual_checks],
        "notes": list(rep.notes),
        "x_norm": float(np.linalg.norm(rep.x)),
        "x_hash": arr_hash(rep.x),
    }
    arrays = {"history": np.asarray(rep.residual_history)}
    if keep_x:
        arrays["x"] = np.asarray(rep.x)
    else:
        arrays["x_head"] = np.asarray(rep.x[:64])
    return d, arrays


def small_cases():
    """Policy / edge cases at desk scale (mirroring the reference test suite)."""
    cases = []

    def add(name, A, b, t, cfg, x0=None, parts=None):
        p = parts if parts is not None else ekcg.contiguous_partition(A.n, t)
        cases.append((name, A, b, x0, p, cfg))

    A = ekcg.gen_poisson2d(12, 12)
    b, _ = ekcg.make_rhs(A, 10)
    add("p12_srecg2_t4_full", A, b, 4, dict(method="sre-cg2", t=4))
    add("p12_srecg2_t4_trunc3", A, b, 4, dict(method="sre-cg2", t=4, retention="trunc", trunc=3))
    add("p12_srecg2_t8_trunc2", A, b, 8, dict(method="sre-cg2", t=8, retention="trunc", trunc=2))
    add("p12_msdo_t4", A, b, 4, dict(method="msdo-cg", t=4))
    add("p12_modmsdo_t4", A, b, 4, dict(method="modified-msdo-cg", t=4))
    add("p12_srecg2_t16_full", A, b, 16, dict(method="sre-cg2", t=16))
    add("p12_srecg2_t32_trunc4", A, b, 32, dict(method="sre-cg2", t=32, retention="trunc", trunc=4))
    A = ekcg.gen_poisson2d(10, 10)
    b, _ = ekcg.make_rhs(A, 11)
    add("p10_srecg_t2", A, b, 2, dict(method="sre-cg", t=2))
    add("p10_srecg2_t2_trunc2", A, b, 2, dict(method="sre-cg2", t=2, retention="trunc", trunc=2))
    b, _ = ekcg.make_rhs(A, 3)
    add("p10_maxiter_t2", A, b, 2, dict(method="sre-cg2", t=2, kmax=4))
    b, _ = ekcg.make_rhs(A, 4)
    add("p10_t1", A, b, 1, dict(method="sre-cg2", t=1))
    rng = np.random.default_rng(12345)
    x0 = rng.standard_normal(A.n)
    add("p10_x0_t4", A, b, 4, dict(method="sre-cg2", t=4), x0=x0)
    A = ekcg.gen_poisson2d(12, 12)
    b, _ = ekcg.make_rhs(A, 12)
    add("p12_restart5_t2", A, b, 2, dict(method="sre-cg2", t=2, retention="restart", restart_j=5))
    A = ekcg.gen_skyscraper(12, 12, contrast=1e4)
    b, _ = ekcg.make_rhs(A, 13)
    add("sky12_restarttol_t2", A, b, 2, dict(method="sre-cg2", t=2, retention="restart-tol",
                                              restart_tol=1e-3))
    A = ekcg.gen_skyscraper(20, 20, contrast=1e6)
    b, _ = ekcg.make_rhs(A, 17)
    add("sky20_stagnation_t2", A, b, 2, dict(method="sre-cg2", t=2, retention="restart", restart_j=5,
                                              kmax=400))
    A = ekcg.gen_poisson2d(16, 16)
    b, _ = ekcg.make_rhs(A, 14)
    add("p16_switch_t4", A, b, 4, dict(method="sre-cg2", t=4, switch_tol=1e-5))
    b, _ = ekcg.make_rhs(A, 42)
    add("p16_switch_trunc4_t4", A, b, 4, dict(method="sre-cg2", t=4, retention="trunc", trunc=4,
                                               switch_tol=1e-4, tol=1e-6))
    A = ekcg.gen_poisson2d(20, 20)
    b, _ = ekcg.make_rhs(A, 43)
    add("p20_trueres25_t2", A, b, 2, dict(method="sre-cg2", t=2, true_residual_every=25))
    A = ekcg.gen_poisson2d(4, 4)
    b = np.zeros(16)
    b[8:] = 1.0
    add("p4_breakdown_t2", A, b, 2, dict(method="sre-cg2", t=2))
    idx = np.arange(12)
    A = ekcg.SparseSpdMatrix.from_coo(12, idx, idx, np.ones(12))
    b = np.random.default_rng(12345).standard_normal(12)
    add("identity12_t4", A, b, 4, dict(method="sre-cg2", t=4))
    A = ekcg.gen_poisson2d(8, 8)
    b = np.zeros(64)
    add("p8_zero_rhs_t2", A, b, 2, dict(method="sre-cg2", t=2))
    A = ekcg.gen_aniso3d(6, 6, 6, 100.0)
    b, _ = ekcg.make_rhs(A, 7)
    owner, p = box_subdomains((6, 6, 6), (2, 2, 2))
    add("aniso6_box222_t8", A, b, 8, dict(method="sre-cg2", t=8, retention="trunc", trunc=3), parts=p)
    return cases


def main():
    skip_cfg2 = "--skip-cfg2" in sys.argv
    meta = {"numpy": np.__version__, "generated": time.strftime("%Y-%m-%d %H:%M:%S"), "cpus": os.cpu_count()}

    # ---- kernel-level vectors ----
    rng = np.random.default_rng(2024)
    kern = {}
    owner = np.array([0, 1, 1, 0, 2, 2, 1], dtype=np.int64)
    p = ekcg.Partition(7, [np.flatnonzero(owner == j) for j in range(3)])
    v = rng.standard_normal(7)
    kern["split_owner"], kern["split_v"], kern["split_W"] = owner, v, p.split(v)
    for tag, n, dens in (("a", 60, 0.05), ("b", 300, 0.02), ("c", 220, 0.6)):
        D = rng.standard_normal((n, n)) * (rng.random((n, n)) < dens)
        D = D + D.T + np.diag(np.abs(D).sum(axis=1) + 1.0)
        rows, cols = np.nonzero(D)
        A = ekcg.SparseSpdMatrix.from_coo(n, rows, cols, D[rows, cols])
        X = rng.standard_normal((n, 70))
        kern[f"spmm_{tag}_rp"], kern[f"spmm_{tag}_ci"], kern[f"spmm_{tag}_v"] = A.row_ptr, A.col_idx, A.values
        kern[f"spmm_{tag}_X"] = X
        kern[f"spmm_{tag}_Y"] = ekcg.spmm(A, X)
        kern[f"spmv_{tag}_y"] = ekcg.spmv(A, X[:, 3].copy())
    B = np.array([[4.0, 2.0], [2.0, 5.0]])
    kern["chol_2x2_B"], kern["chol_2x2_R"] = B, ekcg.cholesky_small(B)
    W = rng.standard_normal((40, 6))
    G = W.T @ W
    kern["chol_rand_B"], kern["chol_rand_R"] = G, ekcg.cholesky_small(G)
    X = rng.standard_normal((50, 6))
    kern["trsm_X"], kern["trsm_R"], kern["trsm_Y"] = X, kern["chol_rand_R"], ekcg.trsm_right_inv(X, kern["chol_rand_R"])
    Y = rng.standard_normal((50, 4))
    kern["gram_X"], kern["gram_Y"], kern["gram_G"] = X, Y, ekcg.gram(X, Y)
    np.savez_compressed(OUT / "kernels.npz", **kern)

    # ---- generator hashes ----
    gens = {}
    for name, A in [
        ("poisson2d_100", ekcg.gen_poisson2d(100, 100)),
        ("poisson3d_16", ekcg.gen_poisson3d(16, 16, 16)),
        ("poisson3d_64", ekcg.gen_poisson3d(64, 64, 64)),
        ("skyscraper2d_12_1e4", ekcg.gen_skyscraper(12, 12, contrast=1e4)),
        ("skyscraper3d_10_11_12", ekcg.gen_skyscraper(10, 11, 12)),
        ("aniso3d_6_100", ekcg.gen_aniso3d(6, 6, 6, 100.0)),
        ("cfg3_16", config_inputs(3, 16)[0]),
        ("cfg3_32", config_inputs(3, 32)[0]),
        ("cfg5_64", config_inputs(5, 64)[0]),
        ("cfg5_256", config_inputs(5, 256)[0]),
    ]:
        gens[name] = {"n": A.n, "nnz": A.nnz, "sha256": csr_hash(A)}
    for (idx, N) in ((1, 100), (2, 16), (2, 64), (3, 16), (3, 32), (5, 64), (5, 256)):
        A, b, xs, part, kw = config_inputs(idx, N)
        gens[f"cfg{idx}_{N}_rhs"] = {"b_sha256": arr_hash(b), "owner_sha256": arr_hash(part.owner())}
    (OUT / "generators.json").write_text(json.dumps(gens, indent=1, sort_keys=True))

    # ---- solves ----
    solves, arrays = {"_meta": meta}, {}

    def run(name, A, b, x0, part, kw, x_star=None, keep_x=True, store_inputs=True):
        cfg = ekcg.SolverConfig(**kw)
        t0 = time.perf_counter()
        _, rep = ekcg.enlarged_solve(A, b, x0=x0, partition=part, cfg=cfg, x_star=x_star)
        dt = time.perf_counter() - t0
        d, arrs = report_dict(rep, keep_x)
        d["cfg"] = kw
        d["wall_s"] = dt
        d["n"] = int(A.n)
        solves[name] = d
        for k, v in arrs.items():
            arrays[f"{name}__{k}"] = v
        if store_inputs:
            arrays[f"{name}__b"] = np.asarray(b)
            arrays[f"{name}__owner"] = np.asarray(part.owner())
            arrays[f"{name}__rp"], arrays[f"{name}__ci"], arrays[f"{name}__vals"] = A.row_ptr, A.col_idx, A.values
            if x0 is not None:
                arrays[f"{name}__x0"] = np.asarray(x0)
        print(f"{name}: {rep.status} it={rep.iterations} wall={dt:.2f}s", flush=True)

    for (name, A, b, x0, part, kw) in small_cases():
        run(name, A, b, x0, part, kw)
    for (idx, N) in ((1, 100), (2, 16), (3, 16), (3, 32), (5, 64)):
        A, b, xs, part, kw = config_inputs(idx, N)
        run(f"cfg{idx}_{N}", A, b, None, part, kw, x_star=xs, keep_x=(A.n <= 40000), store_inputs=False)
    (OUT / "solves.json").write_text(json.dumps(solves, indent=1, sort_keys=True))
    np.savez_compressed(OUT / "solves.npz", **arrays)
    if not skip_cfg2:
        A, b, xs, part, kw = config_inputs(2, 64)
        run("cfg2_64", A, b, None, part, kw, x_star=xs, keep_x=False, store_inputs=False)
        (OUT / "solves.json").write_text(json.dumps(solves, indent=1, sort_keys=True))
        np.savez_compressed(OUT / "solves.npz", **arrays)
    print("done")


if __name__ == "__main__":
    main()
