"""Host readback options for a 537 MB result vector (config-5 x)."""
import time
import numpy as np
import torch
n = 8192 * 8192
x = torch.randn(n, dtype=torch.float64, device="cuda")
cache = torch.empty(n, dtype=torch.float64, pin_memory=True)
def t(name, f, reps=4):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); out = f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(f"{name}: {min(ts)*1e3:.1f} ms (all {[round(v*1e3,1) for v in ts]})", flush=True)
t("x.cpu().numpy()", lambda: x.cpu().numpy())
t("pinned cache + numpy copy", lambda: (cache.copy_(x), cache.numpy().copy())[1])
t("fresh pinned", lambda: torch.empty(n, dtype=torch.float64, pin_memory=True).copy_(x).numpy())
def prefault():
    a = np.empty(n); a.fill(0.0); torch.from_numpy(a).copy_(x); return a
t("np.empty + fill + copy_", prefault)
b = np.random.default_rng(0).standard_normal(n)
t("np.isfinite(b).all()", lambda: np.isfinite(b).all())
bt = torch.from_numpy(b)
t("torch.isfinite(b_cpu).all()", lambda: bool(torch.isfinite(bt).all()))
