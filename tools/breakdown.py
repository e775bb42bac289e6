"""Per-kernel-tag time breakdown of a solve (CUDA events around every tagged launch).

    python tools/breakdown.py --config 3 --kmax 200 [--edge E]

Untagged launches (reduce, small factorizations, finish) show up as the
remainder between the solve's event-timed total and the tagged sum.
"""
import argparse
import json
import sys
from collections import defaultdict
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_19013_b200 as pk  # noqa: E402
from paper_2305_19013_b200.engine import DeviceEngine  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402


class Hook:
    def __init__(self):
        self.used = []
        self.engine = None

    def __call__(self, tag, fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        cur = getattr(self.engine, "_cur", None) or (0, 0, 0)
        self.used.append((tag, cur, e0, e1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--edge", type=int, default=None)
    ap.add_argument("--kmax", type=int, default=None)
    ap.add_argument("--no-fuse", action="store_true")
    ap.add_argument("--once", action="store_true", help="one solve (for ncu launch counting)")
    args = ap.parse_args()
    prob = make_config(args.config, args.edge)
    kw = dict(prob.solver_kwargs)
    if args.kmax:
        kw["kmax"] = args.kmax
    cfg = pk.SolverConfig(**kw)
    op = prob.stencil()
    b = torch.as_tensor(prob.b, device="cuda")
    res = None
    for rep in range(1 if args.once else 2):  # the first solve pays one-time setup
        eng = None
        hook = None
        torch.cuda.empty_cache()
        eng = DeviceEngine(op, prob.partition, cfg)
        eng.no_fuse = args.no_fuse
        hook = Hook()
        hook.engine = eng
        eng.kernel_timer = hook
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        _, rep_ = eng.solve(b)
        s1.record()
        s1.synchronize()
        res = (s0.elapsed_time(s1), hook, rep_)
        hook.engine = None
        del eng, _
    total, hook, rep_ = res
    by = defaultdict(lambda: [0.0, 0])
    for tag, cur, e0, e1 in hook.used:
        if cur[0] <= rep_.iterations:
            ms = e0.elapsed_time(e1)
            by[tag][0] += ms
            by[tag][1] += 1
    by_d = defaultdict(lambda: [0.0, 0])  # the CGS2 kernels per history depth d
    for tag, cur, e0, e1 in hook.used:
        if cur[0] <= rep_.iterations and tag in ("hist_gram", "hist_update"):
            by_d[f"{tag}@d={cur[1]}"][0] += e0.elapsed_time(e1)
            by_d[f"{tag}@d={cur[1]}"][1] += 1
    tagged = sum(v[0] for v in by.values())
    out = {"config": prob.name, "iterations": rep_.iterations, "total_ms": round(total, 2),
           "ms_per_it": round(total / max(rep_.iterations, 1), 4),
           "tags": {k: {"ms": round(v[0], 2), "n": v[1], "share": round(v[0] / total, 3)}
                    for k, v in sorted(by.items(), key=lambda kv: -kv[1][0])},
           "cgs2_ms_per_launch_by_depth": {k: round(v[0] / v[1], 3) for k, v in sorted(by_d.items())},
           "untagged_share": round(1 - tagged / total, 3),
           "model_GBs": rep_.model_bytes / (total / 1e3) / 1e9}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
