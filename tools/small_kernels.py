"""Event-timed back-to-back launches of the small per-iteration kernels
(Pre-CholQR factor, Cholesky inverse, Gram reduction) at m = 16 / 32 / 64.

    python tools/small_kernels.py
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_19013_b200 import _lib  # noqa: E402

dev = "cuda"
st = torch.cuda.current_stream().cuda_stream
ctrl = torch.zeros(_lib.query("ekcg_ctrl_bytes"), dtype=torch.uint8, device=dev)


def timeit(fn, reps=200):
    for _ in range(5):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for m in (16, 32, 64):
    X = torch.randn(4 * m, m, dtype=torch.float64, device=dev)
    G = (X.T @ X).contiguous()
    S = torch.empty_like(G)
    _lib.call("ekcg_start", ctrl.data_ptr(), torch.ones(1, dtype=torch.float64, device=dev).data_ptr(), 1e-30,
              torch.zeros(8, dtype=torch.float64, device=dev).data_ptr(), st)
    ctrl[0:4].view(torch.int32).fill_(1)  # live
    _lib.call("ekcg_cholinv", G.data_ptr(), m, S.data_ptr(), ctrl.data_ptr(), 1, 1e-14, st)
    out = {"m": m, "cholinv_check": float((S.T @ G @ S - torch.eye(m, dtype=torch.float64, device=dev)).abs().max())}
    out["prechol_us"] = timeit(lambda: _lib.call("ekcg_prechol", G.data_ptr(), m, S.data_ptr(), ctrl.data_ptr(), 1,
                                                 1e-14, st))
    out["cholinv_us"] = timeit(lambda: _lib.call("ekcg_cholinv", G.data_ptr(), m, S.data_ptr(), ctrl.data_ptr(), 1,
                                                 1e-14, st))
    for chunks in (148, 444):
        part = torch.randn(chunks * m * m, dtype=torch.float64, device=dev)
        out[f"reduce{chunks}_us"] = timeit(lambda: _lib.call("ekcg_reduce", part.data_ptr(), chunks, m * m,
                                                             G.data_ptr(), None, st))
    print(json.dumps(out), flush=True)
