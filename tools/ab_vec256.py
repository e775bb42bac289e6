"""A/B of 256-bit row loads (ekcg_tune 24) in X^T y and the fused x / r update,
event timed at config sizes, alternating.

    python tools/ab_vec256.py
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_19013_b200 import _lib  # noqa: E402

dev = "cuda"
st = torch.cuda.current_stream().cuda_stream


def t(fn, reps=20):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for m, n in ((16, 64 ** 3), (32, 128 ** 3), (64, 256 ** 3), (64, 8192 * 8192)):
    W = torch.randn(n * m, dtype=torch.float64, device=dev)
    AW = torch.randn(n * m, dtype=torch.float64, device=dev)
    y = torch.randn(n, dtype=torch.float64, device=dev)
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    tab = torch.tensor([W.data_ptr()], dtype=torch.int64, device=dev)
    ch = _lib.query("ekcg_gram_chunks", n, 1, m, 1)
    part = torch.empty(max(ch * m, 1 << 16), dtype=torch.float64, device=dev)
    alpha = torch.randn(m, dtype=torch.float64, device=dev) * 1e-3
    vp = torch.empty(_lib.query("ekcg_vec_chunks", n), dtype=torch.float64, device=dev)
    res = {"m": m, "n": n}
    for name, fn, nbytes in (
            ("gemvt", lambda: _lib.call("ekcg_gram", tab.data_ptr(), m, 1, m, y.data_ptr(), 1, 1, n, part.data_ptr(),
                                        None, st), 8 * n * (m + 1)),
            ("xr", lambda: _lib.call("ekcg_xr_update", W.data_ptr(), m, AW.data_ptr(), m, alpha.data_ptr(), m,
                                     x.data_ptr(), y.data_ptr(), n, vp.data_ptr(), None, st), 8 * n * (2 * m + 4))):
        best = {0: 1e9, 1: 1e9}
        for rep in range(4):
            for v in ((0, 1) if rep % 2 == 0 else (1, 0)):
                _lib.call("ekcg_tune", 24, v)
                best[v] = min(best[v], t(fn))
        res[name] = {"us_128": round(best[0], 1), "us_256": round(best[1], 1),
                     "frac_128": round(nbytes / best[0] / 6548.5e3, 3), "frac_256": round(nbytes / best[1] / 6548.5e3, 3)}
    _lib.call("ekcg_tune", 24, 1)
    print(json.dumps(res), flush=True)
    del W, AW, y, x
    torch.cuda.empty_cache()
