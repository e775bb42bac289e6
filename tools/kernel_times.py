"""Event-timed kernel sweep at config sizes: Gram, block update, stencil, fused stencil kernels.

    python tools/kernel_times.py [m n d ...]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_19013_b200 import _lib  # noqa: E402
from paper_2305_19013_b200.operators import StencilOperator  # noqa: E402

dev = "cuda"
st = torch.cuda.current_stream().cuda_stream
DMMA_TF = 37.1e12
HBM = 6555.5e9


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def sweep(m, shape, d):
    n = 1
    for s in shape:
        n *= s
    out = {}
    Xs = [torch.randn(n * m, dtype=torch.float64, device=dev) for _ in range(d)]
    Y = torch.randn(n * m, dtype=torch.float64, device=dev)
    W = torch.randn(n * m, dtype=torch.float64, device=dev)
    tab = torch.tensor([x.data_ptr() for x in Xs], dtype=torch.int64, device=dev)
    chunks = _lib.query("ekcg_gram_chunks", n, d, m, m)
    part = torch.empty(max(2048 * d * m * m, 1 << 20), dtype=torch.float64, device=dev)
    C = torch.randn(d * m * m, dtype=torch.float64, device=dev) * 0.01
    for gs in ((0, 3) if m == 16 else (0, 1)):
        for tgt in (0,):
            _lib.call("ekcg_tune", 7 if m == 16 else 15, gs)
            _lib.call("ekcg_tune", 2, tgt)
            ch = _lib.query("ekcg_gram_chunks", n, d, m, m)
            part = torch.empty(max(ch * d * m * m, 1 << 20), dtype=torch.float64, device=dev)
            g = timeit(lambda: _lib.call("ekcg_gram", tab.data_ptr(), m, d, m, Y.data_ptr(), m, m, n, part.data_ptr(),
                                         None, st))
            out[f"gram_s{gs}_t{tgt}"] = dict(s=g, GBs=8 * (d + 1) * n * m / g / 1e9, TF=2 * d * m * m * n / g / 1e12)
    _lib.call("ekcg_tune", 7, 10)
    _lib.call("ekcg_tune", 2, 0)
    _lib.call("ekcg_tune", 5, -1)
    for us in ((0, 2, 5, 6, 7) if m == 16 else (0, 10, 11, 12)):
        if m == 16:
            _lib.call("ekcg_tune", 8, us)
        else:  # 0: register-direct kernels; 10 + v: streamed variant v
            _lib.call("ekcg_tune", 15, 1 if us else 0)
            _lib.call("ekcg_tune", 16, max(us - 10, 0))
        u = timeit(lambda: _lib.call("ekcg_block_update", tab.data_ptr(), m, d, m, C.data_ptr(), W.data_ptr(), m,
                                     W.data_ptr(), m, m, 1.0, -1.0, n, None, st))
        out[f"update_s{us}"] = dict(s=u, GBs=8 * (d + 2) * n * m / u / 1e9, TF=2 * d * m * m * n / u / 1e12)
    _lib.call("ekcg_tune", 8, 5)
    _lib.call("ekcg_tune", 15, 1)
    _lib.call("ekcg_tune", 16, 0)
    op = StencilOperator(shape, 1.0)
    Z = torch.empty_like(Y)
    sp = timeit(lambda: op.apply(Y, m, Z, m, m))
    out["stencil"] = dict(s=sp, GBs=16 * n * m / sp / 1e9)
    for k, v in out.items():
        v["hbm_frac"] = v["GBs"] * 1e9 / HBM
        if "TF" in v:
            v["fp64_frac"] = v["TF"] * 1e12 / DMMA_TF
    return out


if __name__ == "__main__" and "--fused" not in sys.argv and "--stencil" not in sys.argv:  # [--wide]
    cases = [(16, (64, 64, 64), 32), (16, (64, 64, 64), 110), (32, (128, 128, 128), 4), (32, (128, 128, 128), 1),
             (64, (256, 256, 128), 3), (64, (256, 256, 256), 2), (64, (256, 256, 256), 1)]
    if len(sys.argv) > 1 and sys.argv[1] == "--wide":
        cases = [c for c in cases if c[0] >= 32]
    res = {}
    for m, shape, d in cases:
        key = f"m{m}_n{'x'.join(map(str, shape))}_d{d}"
        res[key] = sweep(m, shape, d)
        print(key, json.dumps({k: {kk: round(vv, 4) for kk, vv in v.items()} for k, v in res[key].items()}),
              flush=True)
        torch.cuda.empty_cache()
    json.dump(res, open("gpurun_out/kernel_times.json", "w"), indent=1)


def fused_times():
    """Fused stencil kernels at config sizes (one call each, event timed)."""
    from paper_2305_19013_b200.operators import StencilOperator as SO
    import ctypes
    res = {}
    for m, shape in ((16, (64, 64, 64)), (16, (128, 128, 128)), (16, (512, 512))):
        n = 1
        for v in shape:
            n *= v
        op = SO(shape, 1.0)
        X = torch.randn(n * m, dtype=torch.float64, device=dev)
        Y = torch.empty_like(X)
        x = torch.zeros(n, dtype=torch.float64, device=dev)
        r = torch.randn(n, dtype=torch.float64, device=dev)
        alpha = torch.randn(m, dtype=torch.float64, device=dev) * 1e-3
        part = torch.empty(_lib.query("ekcg_fused_partials", n, m), dtype=torch.float64, device=dev)
        cnt = torch.zeros(64, dtype=torch.int32, device=dev)
        ctrl = torch.zeros(_lib.query("ekcg_ctrl_bytes"), dtype=torch.uint8, device=dev)
        ctrl[0] = 1
        G = torch.empty(m * m, dtype=torch.float64, device=dev)
        hist = torch.zeros(16, dtype=torch.float64, device=dev)
        rho2 = torch.zeros(1, dtype=torch.float64, device=dev)
        _lib.call("ekcg_tune", 9, 1)
        _lib.call("ekcg_tune", 13, int(sys.argv[-1]) if sys.argv[-1].isdigit() else 0)
        tg = timeit(lambda: _lib.call("ekcg_stencil_cholinv", op.desc_ref(), X.data_ptr(), m, m, part.data_ptr(),
                                      cnt.data_ptr(), G.data_ptr(), ctrl.data_ptr(), 1, 1e-14, 0, st))
        tx = timeit(lambda: _lib.call("ekcg_stencil_xr", op.desc_ref(), X.data_ptr(), m, Y.data_ptr(), m, m,
                                      alpha.data_ptr(), x.data_ptr(), r.data_ptr(), part.data_ptr(), cnt.data_ptr(),
                                      ctrl.data_ptr(), 1, 10 ** 9, 0, hist.data_ptr(), 0, rho2.data_ptr(), st))
        ts = timeit(lambda: op.apply(X, m, Y, m, m))
        res[f"m{m}"] = {"stencil_cholinv_GBs": 8 * n * m / tg / 1e9, "stencil_xr_GBs": (16 * n * m + 32 * n) / tx / 1e9,
                        "stencil_GBs": 16 * n * m / ts / 1e9}
        print(f"m{m} {shape}", {k: round(v) for k, v in res[f"m{m}"].items()}, flush=True)
    return res


if __name__ == "__main__" and "--fused" in sys.argv:
    fused_times()


def stencil_ab():
    """Plane-marching vs row-parallel stencil kernel (ekcg_tune 3) at config sizes."""
    import numpy as np
    cases = [(16, (64, 64, 64), None), (16, (128, 128, 128), None), (32, (128, 128, 128), None),
             (64, (256, 256, 128), None), (16, (128, 128, 128), "node"), (32, (2048, 2048), None),
             (8, (128, 128, 128), None), (4, (256, 256, 256), None)]
    for m, shape, kap in cases:
        n = int(np.prod(shape))
        kappa = 1.0 if kap is None else np.exp(np.random.default_rng(0).standard_normal(n))
        op = StencilOperator(shape, kappa)
        X = torch.randn(n * m, dtype=torch.float64, device=dev)
        Y = torch.empty_like(X)
        row = {}
        for march in (0, 1):
            _lib.call("ekcg_tune", 3, march)
            for var in ((0, 2, 4, 5, 6) if march and len(shape) == 3 and m % 16 == 0 else (0,)):
                _lib.call("ekcg_tune", 4, var)
                t = timeit(lambda: op.apply(X, m, Y, m, m), reps=10)
                row[f"march{var}" if march else "row"] = round((16 * n * m + op.matrix_bytes()) / t / 1e9)
        _lib.call("ekcg_tune", 4, 0)
        print(f"m{m} {'x'.join(map(str, shape))} {kap or 'const'}", row, flush=True)
        del X, Y, op
        torch.cuda.empty_cache()


if __name__ == "__main__" and "--stencil" in sys.argv:
    stencil_ab()
