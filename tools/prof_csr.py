"""One CSR SpMM of a config operator for ncu: python tools/prof_csr.py config m [kernel choice, ekcg_tune 17]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_19013_b200.operators import CsrOperator  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

c, m = int(sys.argv[1]), int(sys.argv[2])
if len(sys.argv) > 3:
    from paper_2305_19013_b200 import _lib  # noqa: E402
    _lib.call("ekcg_tune", 17, int(sys.argv[3]))
prob = make_config(c, device_rhs=False)
op = CsrOperator(prob.csr(), "cuda")
X = torch.randn(prob.n * m, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
for _ in range(3):
    op.apply(X, m, Y, m, m)
torch.cuda.synchronize()
print("ok")
