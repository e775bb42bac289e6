"""Event-timed hot kernels at config-5-like sizes for library A/B:  python tools/kbench.py LIB.so [n]

Times (best of 5, L2 flushed before each) the m = 64 CGS2 update and Gram at d = 3, the m = 64 triangular
apply, the x/r update and the config-5 tile-field stencil, and checks the update / Gram against torch.
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2305_19013_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib._LIB_PATH = Path(sys.argv[1]).resolve()
edge = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
from paper_2305_19013_b200.problems import make_config  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
dev = torch.device("cuda")
prob = make_config(5, edge, device_rhs=False)
n, m, d = prob.n, 64, 3
g = torch.Generator(device=dev).manual_seed(1)
Qs = [torch.randn(n, m, dtype=torch.float64, device=dev, generator=g) for _ in range(d)]
W = torch.randn(n, m, dtype=torch.float64, device=dev, generator=g)
Wo = torch.empty_like(W)
C = torch.randn(d * m, m, dtype=torch.float64, device=dev, generator=g) * 0.01
tab = torch.tensor([q.data_ptr() for q in Qs], dtype=torch.int64, device=dev)
tabw = torch.tensor([W.data_ptr()], dtype=torch.int64, device=dev)
chunks = _lib.query("ekcg_gram_chunks", n, d, m, m)
part = torch.empty(chunks * d * m * m, dtype=torch.float64, device=dev)
S = torch.triu(torch.randn(m, m, dtype=torch.float64, device=dev, generator=g)).contiguous()
op = prob.stencil(dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=dev)
alpha = torch.randn(m, dtype=torch.float64, device=dev, generator=g) * 1e-3
x = torch.zeros(n, dtype=torch.float64, device=dev)
r = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
vch = _lib.query("ekcg_vec_chunks", n)
vp = torch.empty(vch, dtype=torch.float64, device=dev)


def timed(fn, reps=5):
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


nm = float(n) * m
res = {}
t = timed(lambda: _lib.call("ekcg_block_update", tab.data_ptr(), m, d, m, C.data_ptr(), W.data_ptr(), m,
                            Wo.data_ptr(), m, m, 1.0, -1.0, n, None, st))
res["update_d3"] = {"ms": t, "tflops": 2 * d * m * nm / t / 1e9}
ref = W - sum(Qs[i] @ C[i * m:(i + 1) * m] for i in range(d))
res["update_d3"]["err"] = float((Wo - ref).abs().max() / ref.abs().max())
del ref
t = timed(lambda: _lib.call("ekcg_gram", tab.data_ptr(), m, d, m, W.data_ptr(), m, m, n, part.data_ptr(), None, st))
res["gram_d3"] = {"ms": t, "tflops": 2 * d * m * nm / t / 1e9}
t = timed(lambda: _lib.call("ekcg_tri_apply", tabw.data_ptr(), m, S.data_ptr(), Wo.data_ptr(), m, m, n, None, st))
res["tri"] = {"ms": t, "tbs": 16 * nm / t / 1e9}
t = timed(lambda: _lib.call("ekcg_xr_update", W.data_ptr(), m, Wo.data_ptr(), m, alpha.data_ptr(), m, x.data_ptr(),
                            r.data_ptr(), n, vp.data_ptr(), None, st))
res["xr"] = {"ms": t, "tbs": 8 * (2 * nm + 4 * n) / t / 1e9}
t = timed(lambda: op.apply(W, m, Wo, m, m))
res["stencil"] = {"ms": t, "tbs": 16 * nm / t / 1e9}
print(json.dumps({"lib": Path(_lib._LIB_PATH).name, "n": n, **{k: {a: round(b, 4) if isinstance(b, float) else b
                                                                   for a, b in v.items()} for k, v in res.items()}}))
