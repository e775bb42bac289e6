"""The reference algorithm (oracle port: numpy / OpenBLAS, bitwise the reference's
operations) on the host CPU for each BASELINE config: seconds per iteration over
the first K iterations, at full size where host memory allows, else on a scaled
instance of the same generator (labelled).  One JSON line per config.

    python tools/cpu_configs.py
"""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import ekcg_oracle as orc  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

# (config, edge or None for full size, iterations)
PLAN = [(1, None, 130), (2, None, 12), (3, None, 2), (4, 128, 1), (5, 2048, 1)]

cores = len(os.sched_getaffinity(0))
for idx, edge, iters in PLAN:
    prob = make_config(idx, edge, device_rhs=False)
    A = prob.csr()
    kw = dict(prob.solver_kwargs)
    t = kw.pop("t")
    kw["kmax"] = iters
    t0 = time.perf_counter()
    out = orc.run_oracle(A.row_ptr, A.col_idx, A.values, prob.b, prob.partition.owner(), t, **kw)
    dt = time.perf_counter() - t0
    print(json.dumps({"config": prob.name, "n": prob.n, "scaled": edge is not None, "iterations": out["iterations"],
                      "seconds": round(dt, 2), "s_per_it": round(dt / max(out["iterations"], 1), 4),
                      "status": out["status"], "cores": cores, "impl": "oracle port (numpy/OpenBLAS)"}), flush=True)
