"""Where the e2e (host numpy in/out) solve spends time beyond the device-resident one.

    python tools/e2e_profile.py [--config 2]
"""
import argparse
import cProfile
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_19013_b200 as pk  # noqa: E402
from paper_2305_19013_b200.engine import DeviceEngine  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--kmax", type=int, default=None)
args = ap.parse_args()
prob = make_config(args.config)
kw = dict(prob.solver_kwargs)
if args.kmax:
    kw["kmax"] = args.kmax
cfg = pk.SolverConfig(**kw)
op = prob.stencil()
b_dev = torch.as_tensor(prob.b, device="cuda")
b_host = torch.from_numpy(np.ascontiguousarray(prob.b)).pin_memory()


def dev_solve():
    eng = DeviceEngine(op, prob.partition, cfg)
    return eng.solve(b_dev)


def host_solve():
    return pk.enlarged_solve(prob.stencil(), b_host.numpy(), partition=prob.partition, cfg=cfg)


for f in (dev_solve, host_solve, dev_solve, host_solve):
    f()
torch.cuda.synchronize()
for name, f in (("device", dev_solve), ("host", host_solve)):
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        _, rep = f()
        e1.record()
        e1.synchronize()
        ts.append((e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0), rep.solve_seconds * 1e3))
    print(name, [tuple(round(v, 2) for v in t) for t in ts])
pr = cProfile.Profile()
pr.enable()
host_solve()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
