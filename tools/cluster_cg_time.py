"""Classical CG (method "cg") on small problems: the one-kernel cluster CG (ekcg_cluster_cg) against the
launch-per-phase loop (three host reads per iteration).   python tools/cluster_cg_time.py [--edges 100,200,362]"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_19013_b200 as pk  # noqa: E402
import importlib  # noqa: E402

cg_mod = importlib.import_module("paper_2305_19013_b200.cg")  # the module (the package attribute is the function)
from paper_2305_19013_b200.problems import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--edges", default="100,200,362")
ap.add_argument("--repeats", type=int, default=3)
args = ap.parse_args()
for edge in [int(e) for e in args.edges.split(",")]:
    prob = make_config(1, edge)
    op = prob.stencil()
    b = torch.as_tensor(prob.b, device="cuda")
    cfg = pk.SolverConfig(method="cg", tol=1e-8)
    out = {"n": prob.n}
    for name, cap in (("cluster", 1 << 22), ("launches", 0)):
        cg_mod.CLUSTER_CG_MAX_N = cap
        best = None
        for _ in range(args.repeats):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            x, rep = pk.cg(op, b, cfg=cfg)
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) * 1e3
            if best is None or ms < best[0]:
                best = (ms, rep.iterations, rep.status)
        out[name] = {"call_ms": round(best[0], 3), "iterations": best[1], "status": best[2],
                     "us_per_iteration": round(1e3 * best[0] / max(1, best[1]), 2)}
    print(json.dumps(out), flush=True)
