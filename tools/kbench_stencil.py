"""Event-timed plane-march stencil of a config operator for library A/B (L2 flushed between launches), with a
sha256 of the output:  python tools/kbench_stencil.py LIB.so CONFIG EDGE M"""
import hashlib
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2305_19013_b200 import _lib  # noqa: E402

_lib._LIB_PATH = Path(sys.argv[1]).resolve()
from paper_2305_19013_b200.problems import make_config  # noqa: E402

idx, edge, m = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
prob = make_config(idx, edge, device_rhs=False)
op = prob.stencil("cuda")
g = torch.Generator(device="cuda").manual_seed(3)
X = torch.randn(prob.n * m, dtype=torch.float64, device="cuda", generator=g)
Y = torch.empty_like(X)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
best = 1e30
for _ in range(7):
    flush.fill_(0.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rc = _lib.query("ekcg_spmm_stencil_kernel", 1, op.desc_ref(), X.data_ptr(), m, Y.data_ptr(), m, m, None, st)
    e1.record()
    e1.synchronize()
    assert rc == 0
    best = min(best, e0.elapsed_time(e1))
h = hashlib.sha256(Y.cpu().numpy().tobytes()).hexdigest()[:16]
print(json.dumps({"lib": Path(sys.argv[1]).name, "cfg": idx, "edge": edge, "m": m, "ms": round(best, 4),
                  "tbs": round(16.0 * prob.n * m / best / 1e9, 3), "sha": h}))
