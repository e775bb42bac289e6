"""One block update for ncu: python tools/prof_update.py variant d [m n]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_19013_b200 import _lib  # noqa: E402

var, d = int(sys.argv[1]), int(sys.argv[2])
m = int(sys.argv[3]) if len(sys.argv) > 3 else 16
n = int(sys.argv[4]) if len(sys.argv) > 4 else 262144
st = torch.cuda.current_stream().cuda_stream
Xs = [torch.randn(n * m, dtype=torch.float64, device="cuda") for _ in range(d)]
W = torch.randn(n * m, dtype=torch.float64, device="cuda")
tab = torch.tensor([x.data_ptr() for x in Xs], dtype=torch.int64, device="cuda")
C = torch.randn(d * m * m, dtype=torch.float64, device="cuda") * 0.01
_lib.call("ekcg_tune", 8, var)
for _ in range(3):
    _lib.call("ekcg_block_update", tab.data_ptr(), m, d, m, C.data_ptr(), W.data_ptr(), m, W.data_ptr(), m, m, 1.0,
              -1.0, n, None, st)
torch.cuda.synchronize()
print("ok")
