"""Measure the reference's own reordering floor for every golden solve.

The reference (`ekcg`, run here from /root/reference) is re-run on the
symmetrically permuted system P A P^T, P b with the permuted partition --
the same mathematics with a different floating-point summation order, which
is all any parallel implementation changes.  The max relative deviation of
its residual history from the unpermuted run over k <= 20 is the floor below
which no reordered implementation can be required to agree.  On
well-conditioned systems it is ~1e-15; on the config-5 class and the layered
anisotropic case it is O(0.1-1).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_floors.py

Writes tests/golden/floors.json.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, os.environ.get("EKCG_REFERENCE", "/root/reference/pkg/src"))
import ekcg  # noqa: E402

OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(OUT))
from make_golden import config_inputs  # noqa: E402

K = 20
PERM_SEEDS = (1, 2, 3)


def permute(A, b, owner, perm):
    n = A.n
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    rows = np.repeat(np.arange(n), np.diff(A.row_ptr))
    Ap = ekcg.SparseSpdMatrix.from_coo(n, inv[rows], inv[A.col_idx], A.values)
    own = owner[perm]
    t = int(own.max()) + 1
    return Ap, b[perm], ekcg.Partition(n, [np.flatnonzero(own == j) for j in range(t)])


def rel_dev(a, b):
    n = min(len(a), len(b), K + 1)
    ra, rb = a[:n] / a[0], b[:n] / b[0]
    keep = rb >= 1e-12
    return float(np.max(np.abs(ra[keep] - rb[keep]) / rb[keep])) if keep.any() else 0.0


def main():
    meta = json.loads((OUT / "solves.json").read_text())
    arrays = dict(np.load(OUT / "solves.npz"))
    floors = {}
    for name, d in sorted(meta.items()):
        if name.startswith("_") or d["iterations"] == 0:
            continue
        kw = dict(d["cfg"])
        if name.startswith("cfg"):
            idx, edge = int(name[3]), int(name.split("_")[1])
            A, b, _, part, _ = config_inputs(idx, edge)
            owner = part.owner()
        else:
            rp, ci, vals = arrays[f"{name}__rp"], arrays[f"{name}__ci"], arrays[f"{name}__vals"]
            A = ekcg.SparseSpdMatrix(len(rp) - 1, rp, ci, vals)
            b, owner = arrays[f"{name}__b"], arrays[f"{name}__owner"]
        if kw.get("switch_tol") is not None or kw.get("retention") == "restart-tol":
            kw_run = kw
        else:
            kw_run = dict(kw, kmax=min(K, kw.get("kmax") or K))
        devs = []
        for seed in PERM_SEEDS:
            perm = np.random.default_rng(seed).permutation(A.n)
            Ap, bp, pp = permute(A, b, owner, perm)
            _, rep = ekcg.enlarged_solve(Ap, bp, x0=None if f"{name}__x0" not in arrays
                                         else arrays[f"{name}__x0"][perm], partition=pp,
                                         cfg=ekcg.SolverConfig(**kw_run))
            devs.append(rel_dev(rep.residual_history, arrays[f"{name}__history"]))
        floors[name] = {"max_dev_k20": max(devs), "devs": devs}
        if max(devs) > 1e-6:
            # chaotic class: also record the reordered runs' iteration counts
            its = []
            for seed in PERM_SEEDS:
                perm = np.random.default_rng(seed).permutation(A.n)
                Ap, bp, pp = permute(A, b, owner, perm)
                _, rep = ekcg.enlarged_solve(Ap, bp, partition=pp, cfg=ekcg.SolverConfig(**kw))
                its.append(int(rep.iterations))
            floors[name]["iterations_reordered"] = its
        print(f"{name}: floor {max(devs):.3e} {floors[name].get('iterations_reordered', '')}", flush=True)
    (OUT / "floors.json").write_text(json.dumps(floors, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
