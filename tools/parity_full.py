"""History parity of the device engine with the CPU oracle (the reference
algorithm, pinned bitwise to `ekcg`) over the first K iterations at full
BASELINE sizes (configs 2, 3) and on large scaled instances (configs 4, 5),
on the same inputs.  One JSON line per case: max_k<=K |h_gpu/h0 - h_ref/h0| /
(h_ref/h0).

    python tools/parity_full.py [--k 20] [--cases 2,3,4@128,5@1024]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_19013_b200 as pk  # noqa: E402
from oracle import ekcg_oracle as orc  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=20)
ap.add_argument("--cases", default="2,3,4@128,5@1024")
args = ap.parse_args()
for case in args.cases.split(","):
    idx, _, edge = case.partition("@")
    prob = make_config(int(idx), int(edge) if edge else None, device_rhs=False)
    kw = dict(prob.solver_kwargs)
    kw["kmax"] = args.k
    t0 = time.perf_counter()
    _, rep = pk.enlarged_solve(prob.stencil(), prob.b, partition=prob.partition, cfg=pk.SolverConfig(**kw))
    t_gpu = time.perf_counter() - t0
    A = prob.csr()
    t = kw.pop("t")
    t0 = time.perf_counter()
    ref = orc.run_oracle(A.row_ptr, A.col_idx, A.values, prob.b, prob.partition.owner(), t, **kw)
    t_cpu = time.perf_counter() - t0
    h, g = np.asarray(rep.residual_history), np.asarray(ref["residual_history"])
    n = min(len(h), len(g))
    dev = np.abs(h[:n] / h[0] - g[:n] / g[0]) / (g[:n] / g[0])
    print(json.dumps({"config": prob.name, "n": prob.n, "k": n - 1, "max_rel_dev": float(dev.max()),
                      "dev_at_k": [float(v) for v in dev[:: max(1, (n - 1) // 5)]],
                      "gpu_s": round(t_gpu, 2), "cpu_s": round(t_cpu, 1)}), flush=True)
    del A, ref, rep
    torch.cuda.empty_cache()
