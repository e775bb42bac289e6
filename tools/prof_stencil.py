"""Launch the stencil kernels once each at config-2 size (for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2305_19013_b200 import _lib
from paper_2305_19013_b200.operators import StencilOperator

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
shape = tuple(int(v) for v in sys.argv[2].split("x")) if len(sys.argv) > 2 else (64, 64, 64)
dev = "cuda"
st = torch.cuda.current_stream().cuda_stream
n = 1
for v in shape:
    n *= v
op = StencilOperator(shape, 1.0)
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
for _ in range(2):
    op.apply(X, m, Y, m, m)
    _lib.call("ekcg_stencil_cholinv", op.desc_ref(), X.data_ptr(), m, m, part.data_ptr(), cnt.data_ptr(),
              G.data_ptr(), ctrl.data_ptr(), 1, 1e-14, 0, st)
    _lib.call("ekcg_stencil_xr", op.desc_ref(), X.data_ptr(), m, Y.data_ptr(), m, m, alpha.data_ptr(),
              x.data_ptr(), r.data_ptr(), part.data_ptr(), cnt.data_ptr(), ctrl.data_ptr(), 1, 10 ** 9, 0,
              hist.data_ptr(), 0, rho2.data_ptr(), st)
torch.cuda.synchronize()
print("ok")
