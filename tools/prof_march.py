"""One plain stencil application (march kernel) for ncu: python tools/prof_march.py m nx ny nz [variant] [kappa]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2305_19013_b200 import _lib  # noqa: E402
from paper_2305_19013_b200.operators import StencilOperator  # noqa: E402

m, nx, ny, nz = (int(v) for v in sys.argv[1:5])
var = int(sys.argv[5]) if len(sys.argv) > 5 else 0
kap = sys.argv[6] if len(sys.argv) > 6 else "const"
n = nx * ny * nz
if kap == "tile":
    f = np.exp(np.random.default_rng(0).standard_normal((1, ny // 16, nx // 16)))
    op = StencilOperator((nx, ny, nz), f, tile=(16, 16, nz))
else:
    op = StencilOperator((nx, ny, nz), 1.0)
_lib.call("ekcg_tune", 4, var)
X = torch.randn(n * m, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
for _ in range(3):
    op.apply(X, m, Y, m, m)
torch.cuda.synchronize()
print("ok")
