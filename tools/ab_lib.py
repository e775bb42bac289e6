"""A/B two builds of the kernel library on one config solve, alternating
processes: python tools/ab_lib.py libA.so libB.so [config] [rounds]"""
import json
import statistics
import subprocess
import sys

CHILD = r'''
import sys, json, torch
sys.path.insert(0, ".")
from paper_2305_19013_b200 import _lib
from pathlib import Path
_lib._LIB_PATH = Path(sys.argv[1]).resolve()
import paper_2305_19013_b200 as pk
from paper_2305_19013_b200.engine import DeviceEngine
from paper_2305_19013_b200.problems import make_config
prob = make_config(int(sys.argv[2]))
cfg = pk.SolverConfig(**prob.solver_kwargs)
op = prob.stencil()
b = torch.as_tensor(prob.b, device="cuda")
out = []
for i in range(5):
    eng = DeviceEngine(op, prob.partition, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); eng.solve(b); e1.record(); e1.synchronize()
    del eng
    if i >= 2:
        out.append(e0.elapsed_time(e1))
print(json.dumps(out))
'''

a, b = sys.argv[1], sys.argv[2]
cfg = sys.argv[3] if len(sys.argv) > 3 else "2"
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 4
res = {a: [], b: []}
for _ in range(rounds):
    for lib in (a, b):
        r = subprocess.run([sys.executable, "-c", CHILD, lib, cfg], capture_output=True, text=True)
        res[lib] += json.loads(r.stdout.strip().splitlines()[-1])
for lib, v in res.items():
    print(f"{lib}: median {statistics.median(v):.2f} ms  min {min(v):.2f}  n={len(v)}")
