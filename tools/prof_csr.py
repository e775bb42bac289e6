"""One CSR SpMM of a config operator, launched 3 times (for ncu: --launch-skip 2 --launch-count 1).

    python tools/prof_csr.py CONFIG EDGE M
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2305_19013_b200 as pk  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

idx, edge, m = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
prob = make_config(idx, edge, device_rhs=False)
op = pk.CsrOperator(prob.csr(), "cuda")
X = torch.randn(prob.n, m, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
for _ in range(3):
    op.apply(X, m, Y, m, m)
torch.cuda.synchronize()
print(f"csr spmm cfg{idx}@{edge} m={m}: n={prob.n} nnz={op.nnz}")
