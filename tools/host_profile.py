"""cProfile of the host side of one solve (where the Python enqueue time goes).

    python tools/host_profile.py [--config 1] [--top 30]
"""
import argparse
import cProfile
import pstats
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_19013_b200 as pk  # noqa: E402
from paper_2305_19013_b200.engine import DeviceEngine  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--top", type=int, default=30)
args = ap.parse_args()
prob = make_config(args.config)
cfg = pk.SolverConfig(**prob.solver_kwargs)
op = prob.stencil()
b = torch.as_tensor(prob.b, device="cuda")
for _ in range(3):
    DeviceEngine(op, prob.partition, cfg).solve(b)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
_, rep = DeviceEngine(op, prob.partition, cfg).solve(b)
torch.cuda.synchronize()
pr.disable()
print("iterations", rep.iterations)
pstats.Stats(pr).sort_stats("tottime").print_stats(args.top)
