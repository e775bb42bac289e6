"""A short config solve (kmax iterations) for launch-level profiling: python tools/short_solve.py cfg kmax"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2305_19013_b200 as pk  # noqa: E402
from paper_2305_19013_b200.engine import DeviceEngine  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

idx, kmax = int(sys.argv[1]), int(sys.argv[2])
prob = make_config(idx)
cfg = pk.SolverConfig(**dict(prob.solver_kwargs, kmax=kmax))
op = prob.stencil()
b = torch.as_tensor(prob.b, device="cuda")
for _ in range(2):
    eng = DeviceEngine(op, prob.partition, cfg)
    _, rep = eng.solve(b)
torch.cuda.synchronize()
print("ok", rep.iterations)
