"""A/B of predicted run-ahead batch sizes (DeviceEngine.predict_batches) on whole solves,
alternating, event timed.

    python tools/ab_batches.py [config ...]
"""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_19013_b200 as pk  # noqa: E402
from paper_2305_19013_b200 import _lib  # noqa: E402
from paper_2305_19013_b200.engine import DeviceEngine  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

for c in [int(v) for v in sys.argv[1:]] or [1, 2]:
    prob = make_config(c)
    cfg = pk.SolverConfig(**prob.solver_kwargs)
    op = prob.stencil()
    b = torch.as_tensor(prob.b, device="cuda")
    res = {True: [], False: []}
    launches = {}
    for rep in range(12):
        for pb in ((True, False) if rep % 2 else (False, True)):
            eng = DeviceEngine(op, prob.partition, cfg)
            eng.predict_batches = pb
            torch.cuda.synchronize()
            l0 = _lib.query("ekcg_launch_count")
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _, r = eng.solve(b)
            e1.record()
            e1.synchronize()
            if rep >= 2:
                res[pb].append(e0.elapsed_time(e1))
            launches[pb] = _lib.query("ekcg_launch_count") - l0
            del eng
    print(json.dumps({"config": c, "iterations": r.iterations,
                      "ms_predicted": round(statistics.median(res[True]), 3),
                      "ms_doubling": round(statistics.median(res[False]), 3),
                      "launches_predicted": launches[True], "launches_doubling": launches[False]}), flush=True)
