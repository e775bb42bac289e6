"""GPU idle time inside one solve: kernel intervals from torch.profiler (CUPTI),
the gaps between consecutive kernels, and where the largest gaps sit.

    python tools/idle_gaps.py [--config 2]
"""
import argparse
import json
import sys
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_19013_b200 as pk  # noqa: E402
from paper_2305_19013_b200.engine import DeviceEngine  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
args = ap.parse_args()
prob = make_config(args.config)
cfg = pk.SolverConfig(**prob.solver_kwargs)
op = prob.stencil()
b = torch.as_tensor(prob.b, device="cuda")


def solve():
    eng = DeviceEngine(op, prob.partition, cfg)
    _, rep = eng.solve(b)
    return rep


for _ in range(2):
    solve()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rep = solve()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.device_resource_id is not None]
k = sorted(((e.time_range.start, e.time_range.end, e.name) for e in ev if "memcpy" not in e.name.lower()
            and "memset" not in e.name.lower()), key=lambda t: t[0])
busy = sum(e - s for s, e, _ in k)
span = k[-1][1] - k[0][0]
gaps = [(k[i + 1][0] - k[i][1], i) for i in range(len(k) - 1)]
pos = [g for g in gaps if g[0] > 0]
big = sorted(pos, reverse=True)[:12]
out = json.dumps({"iterations": rep.iterations, "kernels": len(k), "span_ms": span / 1e3, "busy_ms": busy / 1e3,
                  "idle_ms": sum(g for g, _ in pos) / 1e3,
                  "idle_over_5us_ms": sum(g for g, _ in pos if g > 5) / 1e3,
                  "largest_gaps_us": [(round(g, 1), k[i][2][:40], k[i + 1][2][:40], i) for g, i in big]}, indent=1)
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/idle_gaps.json").write_text(out)
print(out)
