"""A/B of stencil builds: python tools/probe_stencil2.py LIB.so  (config-5 2-D and config-3 3-D fields;
config 3 with and without the per-node coefficient table).  Prints ms and a checksum for bitwise A/B."""
import hashlib
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2305_19013_b200 import _lib  # noqa: E402

_lib._LIB_PATH = Path(sys.argv[1]).resolve()
from paper_2305_19013_b200.problems import make_config  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
CASES = ((5, 8192, 64), (3, 128, 32), (4, 256, 64), (4, 256, 16), (2, 64, 16)) if "--all" in sys.argv else \
    ((5, 8192, 64), (3, 128, 32))
for idx, edge, m in CASES:
    prob = make_config(idx, edge, device_rhs=False)
    op = prob.stencil("cuda")
    g = torch.Generator(device="cuda").manual_seed(3)
    X = torch.randn(prob.n * m, dtype=torch.float64, device="cuda", generator=g)
    Y = torch.empty_like(X)
    for table in ((True, False) if op.coef is not None else (False,)):
        saved = op._desc.coef
        if not table:
            op._desc.coef = None
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            op.apply(X, m, Y, m, m)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        h = hashlib.sha256(Y.cpu().numpy().tobytes()).hexdigest()[:16]
        op._desc.coef = saved
        print(f"{Path(sys.argv[1]).name} cfg{idx}@{edge} m={m} table={table}: {best:.3f} ms, "
              f"{16 * prob.n * m / best / 1e9:.2f} TB/s, sha {h}", flush=True)
    del X, Y, op
    torch.cuda.empty_cache()
