"""Event-timed CSR SpMM of a config operator for library A/B (L2 flushed, best of 7, bitwise checksum):
    python tools/kbench_csr.py LIB.so CONFIG EDGE M"""
import hashlib
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2305_19013_b200 import _lib  # noqa: E402

_lib._LIB_PATH = Path(sys.argv[1]).resolve()
import paper_2305_19013_b200 as pk  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

idx, edge, m = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
prob = make_config(idx, edge, device_rhs=False)
op = pk.CsrOperator(prob.csr(), "cuda")
g = torch.Generator(device="cuda").manual_seed(2)
X = torch.randn(prob.n, m, dtype=torch.float64, device="cuda", generator=g)
Y = torch.empty_like(X)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
best = 1e30
for _ in range(7):
    flush.fill_(0.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    op.apply(X, m, Y, m, m)
    e1.record()
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1))
alg = 16.0 * prob.n * m + op.matrix_bytes()
print(json.dumps({"lib": Path(sys.argv[1]).name, "config": idx, "edge": edge, "m": m, "ms": round(best, 4),
                  "alg_TBs": round(alg / best / 1e9, 3), "sha": hashlib.sha256(Y.cpu().numpy().tobytes()).hexdigest()[:16]}))
