"""Per-iteration device time of a config solve (one CUDA event per iteration) vs host enqueue time.

    python tools/iter_profile.py [config]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2305_19013_b200 as pk  # noqa: E402
from paper_2305_19013_b200.engine import DeviceEngine  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prob = make_config(idx)
cfg = pk.SolverConfig(**prob.solver_kwargs)
op = prob.stencil()
b = torch.as_tensor(prob.b, device="cuda")
import os
from paper_2305_19013_b200 import _lib  # noqa: E402
if os.environ.get("PDL") is not None:
    _lib.call("ekcg_tune", 14, int(os.environ["PDL"]))
orig = DeviceEngine._enqueue_iteration
for rep in range(3):
    evs, host = [], []

    def wrapped(self, k, tol1):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        evs.append((k, e))
        t0 = time.perf_counter()
        orig(self, k, tol1)
        host.append(time.perf_counter() - t0)

    DeviceEngine._enqueue_iteration = wrapped
    eng = DeviceEngine(op, prob.partition, cfg)
    import os
    if os.environ.get("FUSE") is not None:
        eng.fuse = set(f for f in os.environ["FUSE"].split(",") if f)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    s0.record()
    _, rep_ = eng.solve(b)
    s1.record()
    s1.synchronize()
    wall = time.perf_counter() - w0
    DeviceEngine._enqueue_iteration = orig
    total = s0.elapsed_time(s1)
    its = [(k, evs[i][1].elapsed_time(evs[i + 1][1])) for i, (k, _) in enumerate(evs[:-1])]
    first = s0.elapsed_time(evs[0][1])
    print(f"rep {rep}: total {total:.1f} ms wall {wall*1e3:.1f} ms iters {rep_.iterations} setup->it1 {first:.2f} ms "
          f"host enqueue sum {sum(host)*1e3:.1f} ms (mean {sum(host)/len(host)*1e6:.0f} us)")
    if rep == 2:
        for k, ms in its[:30:3] + its[30::10]:
            print(f"  it {k}: {ms*1e3:.0f} us")
        print("  sum iters 1..20:", round(sum(ms for k, ms in its[:20]), 2), "ms; 20..end:", round(sum(ms for k, ms in its[20:]), 2))
