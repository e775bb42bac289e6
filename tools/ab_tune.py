"""A/B an ekcg_tune knob on one config solve, alternating processes.

    python tools/ab_tune.py KEY VALUE_A VALUE_B [config] [rounds] [kmax]
"""
import json
import statistics
import subprocess
import sys

CHILD = r'''
import sys, json, torch
sys.path.insert(0, ".")
from paper_2305_19013_b200 import _lib
import paper_2305_19013_b200 as pk
from paper_2305_19013_b200.engine import DeviceEngine
from paper_2305_19013_b200.problems import make_config
_lib.call("ekcg_tune", int(sys.argv[1]), int(sys.argv[2]))
prob = make_config(int(sys.argv[3]))
kw = dict(prob.solver_kwargs)
if int(sys.argv[4]) > 0:
    kw["kmax"] = int(sys.argv[4])
cfg = pk.SolverConfig(**kw)
op = prob.stencil()
b = torch.as_tensor(prob.b, device="cuda")
out = []
for i in range(4):
    eng = DeviceEngine(op, prob.partition, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); _, rep = eng.solve(b); e1.record(); e1.synchronize()
    del eng
    if i >= 1:
        out.append(e0.elapsed_time(e1) / rep.iterations)
print(json.dumps(out))
'''

key, va, vb = sys.argv[1], sys.argv[2], sys.argv[3]
cfg = sys.argv[4] if len(sys.argv) > 4 else "2"
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 3
kmax = sys.argv[6] if len(sys.argv) > 6 else "0"
res = {va: [], vb: []}
for _ in range(rounds):
    for v in (va, vb):
        r = subprocess.run([sys.executable, "-c", CHILD, key, v, cfg, kmax], capture_output=True, text=True)
        try:
            res[v] += json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            print(r.stderr[-2000:])
            raise
for v, ts in res.items():
    print(f"tune {key}={v}: median {statistics.median(ts):.4f} ms/iteration  min {min(ts):.4f}  n={len(ts)}")
