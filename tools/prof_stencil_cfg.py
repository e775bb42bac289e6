"""The plane-march stencil of a config operator (forced form 1), launched 3 times, for ncu
(--launch-skip 2 --launch-count 1).   python tools/prof_stencil_cfg.py CONFIG EDGE M"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2305_19013_b200 import _lib  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

idx, edge, m = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
prob = make_config(idx, edge, device_rhs=False)
op = prob.stencil("cuda")
X = torch.randn(prob.n * m, dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    assert _lib.query("ekcg_spmm_stencil_kernel", 1, op.desc_ref(), X.data_ptr(), m, Y.data_ptr(), m, m, None,
                      st) == 0
torch.cuda.synchronize()
print(f"plane march cfg{idx}@{edge} m={m}")
