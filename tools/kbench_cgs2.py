"""Event-timed CGS2 update / Gram at (n, m, d) for library A/B:
    python tools/kbench_cgs2.py LIB.so n m d [inplace]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2305_19013_b200 import _lib  # noqa: E402

_lib._LIB_PATH = Path(sys.argv[1]).resolve()
n, m, d = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
inplace = len(sys.argv) > 5
st = torch.cuda.current_stream().cuda_stream
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1)
Qs = [torch.randn(n, m, dtype=torch.float64, device=dev, generator=g) for _ in range(d)]
W = torch.randn(n, m, dtype=torch.float64, device=dev, generator=g)
W0 = W.clone()
Wo = W if inplace else torch.empty_like(W)
C = torch.randn(d * m, m, dtype=torch.float64, device=dev, generator=g) * 0.01
tab = torch.tensor([q.data_ptr() for q in Qs], dtype=torch.int64, device=dev)
chunks = _lib.query("ekcg_gram_chunks", n, d, m, m)
part = torch.empty(chunks * d * m * m, dtype=torch.float64, device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=dev)


def timed(fn, reps=7):
    best = 1e30
    for _ in range(reps):
        if inplace:
            W.copy_(W0)
        flush.fill_(0.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


nm = float(n) * m
t_u = timed(lambda: _lib.call("ekcg_block_update", tab.data_ptr(), m, d, m, C.data_ptr(), W.data_ptr(), m,
                              Wo.data_ptr(), m, m, 1.0, -1.0, n, None, st))
ref = W0 - sum(Qs[i] @ C[i * m:(i + 1) * m] for i in range(d))
err = float((Wo - ref).abs().max() / ref.abs().max())
t_g = timed(lambda: _lib.call("ekcg_gram", tab.data_ptr(), m, d, m, W0.data_ptr(), m, m, n, part.data_ptr(), None,
                              st))
print(json.dumps({"lib": Path(_lib._LIB_PATH).name, "n": n, "m": m, "d": d,
                  "update": {"ms": round(t_u, 4), "tflops": round(2 * d * m * nm / t_u / 1e9, 2),
                             "tbs": round(8 * (d + 2) * nm / t_u / 1e9, 3), "err": err},
                  "gram": {"ms": round(t_g, 4), "tflops": round(2 * d * m * nm / t_g / 1e9, 2),
                           "tbs": round(8 * (d + 1) * nm / t_g / 1e9, 3)}}))
