"""Back-to-back launch cost on one stream: trivial kernels vs the iteration's small kernels."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_19013_b200 import _lib  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
a = torch.ones(1024, dtype=torch.float64, device="cuda")
b = torch.ones(1024, dtype=torch.float64, device="cuda")
o = torch.empty(1024, dtype=torch.float64, device="cuda")
ctrl = torch.zeros(_lib.query("ekcg_ctrl_bytes"), dtype=torch.uint8, device="cuda")
ctrl[0] = 1
G = torch.eye(16, dtype=torch.float64, device="cuda").reshape(-1) * 4.0
S = torch.empty(256, dtype=torch.float64, device="cuda")


def timeit(fn, reps=2000):
    for _ in range(50):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for mode in (0, 1, 2):
    _lib.call("ekcg_tune", 14, mode)
    print(f"sub n=1024 pdl={mode} (us/launch):", round(timeit(lambda: _lib.call("ekcg_sub", a.data_ptr(), b.data_ptr(), o.data_ptr(), 1024, None, st)), 2))
_lib.call("ekcg_tune", 14, 0)
print("prechol m=16 (us/launch):", round(timeit(lambda: _lib.call("ekcg_prechol", G.data_ptr(), 16, S.data_ptr(), ctrl.data_ptr(), 1, 1e-14, st)), 2))
print("cholinv m=16 (us/launch):", round(timeit(lambda: _lib.call("ekcg_cholinv", G.data_ptr(), 16, S.data_ptr(), ctrl.data_ptr(), 1, 1e-14, st)), 2))
# host-side launch rate alone (python + ctypes), no sync
import time
t0 = time.perf_counter()
for _ in range(2000):
    _lib.call("ekcg_sub", a.data_ptr(), b.data_ptr(), o.data_ptr(), 1024, None, st)
t1 = time.perf_counter()
torch.cuda.synchronize()
print("host enqueue (us/launch):", round((t1 - t0) / 2000 * 1e6, 2))
