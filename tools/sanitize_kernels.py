"""Every TMA / mbarrier ring kernel once, at sizes that give several co-resident CTAs per SM and
several ring wraps, for compute-sanitizer (racecheck / synccheck / memcheck), and each result checked
against torch so a sanitizer run also says whether the numbers were right.

    compute-sanitizer --tool racecheck python tools/sanitize_kernels.py

Kernels: the streamed m = 16 Gram (d = 1: one block per CTA, 3 CTAs per SM; d = 5: 4 blocks per CTA) and
update (stream.cu), the streamed m = 32 Gram and update (stream_wide.cu), the plane-march stencil in 3-D and
2-D with kappa tile fields (stencil_march.cu), the fused m = 16 plane marches (stencil + Gram + factor,
stencil + x/r update), and the pipelined CSR SpMM.
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2305_19013_b200 import _lib  # noqa: E402
from paper_2305_19013_b200.operators import StencilOperator  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

DEV = torch.device("cuda", 0)
st = torch.cuda.current_stream().cuda_stream
rng = np.random.default_rng(0)
fails = []


def check(name, got, ref, tol=1e-12):
    err = (got - ref).abs().max().item() / max(ref.abs().max().item(), 1e-300)
    print(f"{name}: rel err {err:.2e}", flush=True)
    if not err <= tol:
        fails.append(name)


def gram(Xs, Y, m):
    n = Y.shape[0]
    d = len(Xs)
    tab = torch.tensor([x.data_ptr() for x in Xs], dtype=torch.int64, device=DEV)
    chunks = _lib.query("ekcg_gram_chunks", n, d, m, m)
    part = torch.empty(chunks * d * m * m, dtype=torch.float64, device=DEV)
    G = torch.empty(d * m * m, dtype=torch.float64, device=DEV)
    _lib.call("ekcg_gram", tab.data_ptr(), m, d, m, Y.data_ptr(), m, m, n, part.data_ptr(), None, st)
    _lib.call("ekcg_reduce", part.data_ptr(), chunks, d * m * m, G.data_ptr(), None, st)
    return G.view(d, m, m)


def update(Qs, C, W, m):
    n = W.shape[0]
    tab = torch.tensor([q.data_ptr() for q in Qs], dtype=torch.int64, device=DEV)
    out = W.clone()
    _lib.call("ekcg_block_update", tab.data_ptr(), m, len(Qs), m, C.data_ptr(), out.data_ptr(), m, out.data_ptr(), m,
              m, 1.0, -1.0, n, None, st)
    return out


for m, n in ((16, 300_000), (32, 200_000)):
    for d in (1, 5):
        Xs = [torch.randn(n, m, dtype=torch.float64, device=DEV) for _ in range(d)]
        Y = torch.randn(n, m, dtype=torch.float64, device=DEV)
        G = gram(Xs, Y, m)
        check(f"gram m={m} d={d}", G, torch.stack([x.T @ Y for x in Xs]))
        C = torch.randn(d * m, m, dtype=torch.float64, device=DEV) * 0.1
        W = update(Xs, C, Y, m)
        check(f"update m={m} d={d}", W, Y - sum(Xs[i] @ C[i * m:(i + 1) * m] for i in range(d)))

for idx, edge, m in ((3, 64, 32), (5, 512, 64), (2, 64, 16)):
    prob = make_config(idx, edge)
    op = prob.stencil(DEV)
    A = prob.csr()
    X = torch.randn(prob.n, m, dtype=torch.float64, device=DEV)
    Y = torch.empty_like(X)
    assert _lib.query("ekcg_spmm_stencil_kernel", 1, op.desc_ref(), X.data_ptr(), m, Y.data_ptr(), m, m, None,
                      st) == 0
    rows = torch.from_numpy(np.repeat(np.arange(prob.n), np.diff(A.row_ptr))).to(DEV)
    cols = torch.from_numpy(A.col_idx).to(DEV)
    vals = torch.from_numpy(A.values).to(DEV)
    ref = torch.zeros_like(X).index_add_(0, rows, vals[:, None] * X[cols])
    check(f"plane march cfg{idx}@{edge} m={m}", Y, ref)
    rp, ci = torch.from_numpy(A.row_ptr).to(DEV), torch.from_numpy(A.col_idx.astype(np.int32)).to(DEV)
    Yc = torch.empty_like(X)
    assert _lib.query("ekcg_spmm_csr_kernel", 1, rp.data_ptr(), ci.data_ptr(), vals.data_ptr(), X.data_ptr(), m,
                      Yc.data_ptr(), m, prob.n, m, None, st) == 0
    check(f"csr pipelined cfg{idx}@{edge} m={m}", Yc, ref)
    if m == 16:  # fused plane marches (m = 16, above the march threshold)
        n = prob.n
        part = torch.empty(_lib.query("ekcg_fused_partials", n, m), dtype=torch.float64, device=DEV)
        cnt = torch.zeros(64, dtype=torch.int32, device=DEV)
        ctrl = torch.zeros(_lib.query("ekcg_ctrl_bytes"), dtype=torch.uint8, device=DEV)
        ctrl[0] = 1
        S = torch.empty(m * m, dtype=torch.float64, device=DEV)
        Xo = torch.linalg.qr(X)[0].contiguous()  # well-conditioned columns
        _lib.call("ekcg_stencil_cholinv", op.desc_ref(), Xo.data_ptr(), m, m, part.data_ptr(), cnt.data_ptr(),
                  S.data_ptr(), ctrl.data_ptr(), 1, 1e-14, 1, st)
        Gaw = Xo.T @ (torch.zeros_like(Xo).index_add_(0, rows, vals[:, None] * Xo[cols]))
        Rinv = S.view(m, m)
        check("fused march A-CholQR (S^T G S = I)", Rinv.T @ (0.5 * (Gaw + Gaw.T)) @ Rinv,
              torch.eye(m, dtype=torch.float64, device=DEV), 1e-10)
        alpha = torch.randn(m, dtype=torch.float64, device=DEV) * 1e-3
        x = torch.zeros(n, dtype=torch.float64, device=DEV)
        r = torch.randn(n, dtype=torch.float64, device=DEV)
        r0 = r.clone()
        AW = torch.empty_like(X)
        hist = torch.zeros(16, dtype=torch.float64, device=DEV)
        rho2 = torch.zeros(1, dtype=torch.float64, device=DEV)
        _lib.call("ekcg_stencil_xr", op.desc_ref(), X.data_ptr(), m, AW.data_ptr(), m, m, alpha.data_ptr(),
                  x.data_ptr(), r.data_ptr(), part.data_ptr(), cnt.data_ptr(), ctrl.data_ptr(), 1, 100, 0,
                  hist.data_ptr(), 0,
                  rho2.data_ptr(), st)
        check("fused march A W", AW, ref)
        check("fused march x/r update", r, r0 - ref @ alpha)
torch.cuda.synchronize()
print("FAILED: " + ", ".join(fails) if fails else "all kernels correct", flush=True)
sys.exit(1 if fails else 0)
