"""Stencil SpMM bandwidth (16 n m bytes per application / event time) for the
config operators and a constant-kappa operator of the same shape.

    python tools/stencil_bw.py [--configs 2,3,4,5]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2305_19013_b200.operators import StencilOperator  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="2,3,4,5")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--variants", default="0", help="plane-march variants (ekcg_tune 4) to time")
ap.add_argument("--csr", action="store_true", help="also time the CSR SpMM of the same operator")
args = ap.parse_args()


def bw(op, m, reps):
    n = op.n
    X = torch.randn(n * m, dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    for _ in range(2):
        op.apply(X, m, Y, m, m)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        op.apply(X, m, Y, m, m)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    del X, Y
    return round(ms, 4), round(16.0 * n * m / (ms / 1e3) / 1e9, 1)


for c in (int(v) for v in args.configs.split(",")):
    prob = make_config(c, device_rhs=False)
    op = prob.stencil()
    widths = {2: [16], 3: [32, 16], 4: [16, 64], 5: [64]}[c]
    const = StencilOperator(op.shape, 1.0)
    from paper_2305_19013_b200 import _lib
    for m in widths:
        if op.n * m * 16 > 100e9:
            continue
        for v in (int(x) for x in args.variants.split(",")):
            _lib.call("ekcg_tune", 4, v)
            print(json.dumps({"config": c, "m": m, "variant": v, "field": op.field is not None,
                              "op": bw(op, m, args.reps), "const_kappa": bw(const, m, args.reps)}), flush=True)
        _lib.call("ekcg_tune", 4, 0)
        if args.csr:
            from paper_2305_19013_b200.operators import CsrOperator
            A = prob.csr()
            cop = CsrOperator(A, "cuda")
            for vec, w256 in ((3, 1), (3, 0), (1, 1), (2, 1), (0, 1)):
                _lib.call("ekcg_tune", 17, vec)
                _lib.call("ekcg_tune", 22, w256)
                ms, _ = bw(cop, m, args.reps)
                nbytes = 16.0 * op.n * m + 12.0 * A.nnz + 8.0 * (op.n + 1)
                print(json.dumps({"config": c, "m": m, "csr_vec": vec, "w256": w256, "csr_ms": ms,
                                  "csr_GBs": round(nbytes / (ms / 1e3) / 1e9, 1)}), flush=True)
            _lib.call("ekcg_tune", 17, 3)
            del cop, A
