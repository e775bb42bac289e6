"""CGS2 Gram / update rate against the number of retained blocks d at m = 16,
64^3 rows (the bench workload), default kernel choices, event timed, L2 flushed.

    python tools/dsweep.py [d ...]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_19013_b200 import _lib  # noqa: E402

dev, m, n = "cuda", 16, 64 ** 3
st = torch.cuda.current_stream().cuda_stream
HBM = 6548.5e9
ds = [int(v) for v in sys.argv[1:] if v.isdigit()] or [2, 4, 8, 16, 32, 64, 110]
Xs = [torch.randn(n * m, dtype=torch.float64, device=dev) for _ in range(max(ds))]
Y = torch.randn(n * m, dtype=torch.float64, device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)


def timeit(fn, reps=10):
    fn()
    tot = 0.0
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps / 1e3


for d in ds:
    tab = torch.tensor([x.data_ptr() for x in Xs[:d]], dtype=torch.int64, device=dev)
    ch = _lib.query("ekcg_gram_chunks", n, d, m, m)
    part = torch.empty(max(ch * d * m * m, 1 << 16), dtype=torch.float64, device=dev)
    C = torch.randn(d * m * m, dtype=torch.float64, device=dev) * 0.01
    G = torch.empty(d * m * m, dtype=torch.float64, device=dev)
    tg = timeit(lambda: _lib.call("ekcg_gram", tab.data_ptr(), m, d, m, Y.data_ptr(), m, m, n, part.data_ptr(), None,
                                  st))
    tr = timeit(lambda: _lib.call("ekcg_reduce", part.data_ptr(), ch, d * m * m, G.data_ptr(), None, st))
    tu = timeit(lambda: _lib.call("ekcg_block_update", tab.data_ptr(), m, d, m, C.data_ptr(), Y.data_ptr(), m,
                                  Y.data_ptr(), m, m, 1.0, -1.0, n, None, st))
    bg, bu = 8 * (d + 1) * n * m, 8 * (d + 2) * n * m
    row = {"d": d, "gram_us": round(tg * 1e6, 1), "gram_frac": round(bg / tg / HBM, 3),
           "reduce_us": round(tr * 1e6, 1), "chunks": ch,
           "update_us": round(tu * 1e6, 1), "update_frac": round(bu / tu / HBM, 3)}
    if "--variants" in sys.argv:
        for v in range(1, 11):
            _lib.call("ekcg_tune", 7, v)
            chv = _lib.query("ekcg_gram_chunks", n, d, m, m)
            pv = torch.empty(max(chv * d * m * m, 1 << 16), dtype=torch.float64, device=dev)
            t = timeit(lambda: _lib.call("ekcg_gram", tab.data_ptr(), m, d, m, Y.data_ptr(), m, m, n, pv.data_ptr(),
                                         None, st))
            row[f"g{v}"] = round(bg / t / HBM, 3)
        _lib.call("ekcg_tune", 7, 10)
        for v in range(1, 8):
            _lib.call("ekcg_tune", 8, v)
            t = timeit(lambda: _lib.call("ekcg_block_update", tab.data_ptr(), m, d, m, C.data_ptr(), Y.data_ptr(), m,
                                         Y.data_ptr(), m, m, 1.0, -1.0, n, None, st))
            row[f"u{v}"] = round(bu / t / HBM, 3)
        _lib.call("ekcg_tune", 8, 5)
    print(json.dumps(row), flush=True)
