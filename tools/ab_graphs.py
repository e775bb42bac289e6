"""Config 1 (and 2) solve time with and without CUDA-graph replay of steady-state iterations.

    python tools/ab_graphs.py [--config 1] [--reps 5]
"""
import argparse
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_19013_b200 as pk  # noqa: E402
from paper_2305_19013_b200.engine import DeviceEngine  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--prechol", action="store_true", help="also fuse update2 + Graw + Pre-CholQR")
args = ap.parse_args()
prob = make_config(args.config)
cfg = pk.SolverConfig(**prob.solver_kwargs)
op = prob.stencil()
b = torch.as_tensor(prob.b, device="cuda")
for graphs in (False, True, False, True):
    ts = []
    for _ in range(args.reps):
        eng = DeviceEngine(op, prob.partition, cfg)
        eng.use_graphs = graphs
        if args.prechol:
            eng.fuse = eng.fuse | {"prechol"}
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x, rep = eng.solve(b)
        e1.record()
        e1.synchronize()
        ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3, rep.iterations))
    best = min(ts)
    print(f"graphs={graphs}: best {best[0]:.2f} ms device ({best[1]:.2f} ms wall), {best[2]} iterations, "
          f"{best[2] / best[0] * 1e3:.0f} it/s; all {[round(t[0], 2) for t in ts]}", flush=True)
