"""Event-timed W^T W (and W^T Z) at (n, m) for library A/B:  python tools/kbench_gram_self.py LIB.so n m"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2305_19013_b200 import _lib  # noqa: E402

_lib._LIB_PATH = Path(sys.argv[1]).resolve()
n, m = int(sys.argv[2]), int(sys.argv[3])
st = torch.cuda.current_stream().cuda_stream
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1)
W = torch.randn(n, m, dtype=torch.float64, device=dev, generator=g)
Z = torch.randn(n, m, dtype=torch.float64, device=dev, generator=g)
tab = torch.tensor([W.data_ptr()], dtype=torch.int64, device=dev)
chunks = _lib.query("ekcg_gram_chunks", n, 1, m, m)
part = torch.empty(chunks * m * m, dtype=torch.float64, device=dev)
G = torch.empty(m * m, dtype=torch.float64, device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=dev)


def timed(fn, reps=7):
    best = 1e30
    for _ in range(reps):
        flush.fill_(0.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


out = {"lib": Path(sys.argv[1]).name, "n": n, "m": m}
for name, Y in (("self", W), ("other", Z)):
    t = timed(lambda: _lib.call("ekcg_gram", tab.data_ptr(), m, 1, m, Y.data_ptr(), m, m, n, part.data_ptr(), None, st))
    _lib.call("ekcg_reduce", part.data_ptr(), chunks, m * m, G.data_ptr(), None, st)
    ref = W.T @ Y
    err = float((G.view(m, m) - ref).abs().max() / ref.abs().max())
    out[name] = {"ms": round(t, 4), "tflops_full": round(2.0 * m * m * n / t / 1e9, 2),
                 "read_tbs": round((1 if Y is W else 2) * 8.0 * n * m / t / 1e9, 3), "err": err}
print(json.dumps(out))
