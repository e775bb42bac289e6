"""Which stencil kernel the automatic form takes at config-5 edges, and its time (CUDA events)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2305_19013_b200 import _lib  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
for edge in (1024, 4096, 8192):
    prob = make_config(5, edge, device_rhs=False)
    op = prob.stencil("cuda")
    m = 64
    X = torch.randn(prob.n * m, dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    for form in (1, 2, 0):
        rc = _lib.query("ekcg_spmm_stencil_kernel", form, op.desc_ref(), X.data_ptr(), m, Y.data_ptr(), m, m, None, st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            _lib.query("ekcg_spmm_stencil_kernel", form, op.desc_ref(), X.data_ptr(), m, Y.data_ptr(), m, m, None, st)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 5
        gb = 16.0 * prob.n * m / 1e9
        print(f"edge {edge} form {form}: rc {rc}, {ms:.3f} ms, {gb / ms:.2f} TB/s", flush=True)
    del X, Y
    torch.cuda.empty_cache()
