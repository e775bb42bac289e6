"""Stress test of the TMA / mbarrier ring kernels (compute-sanitizer is closed on this GPU pool).

Every ring kernel -- streamed m = 16 / 32 Gram and update, the 3-D and 2-D
plane-march stencils, the fused m = 16 march -- is launched 25 times while a
second stream keeps a varying share of the SMs busy with unrelated fp64 GEMMs,
so CTAs land on SMs in changing numbers and orders.  A missing barrier, a slot
refilled before its consumers finished (the round-1 cross-proxy race), or a
phase-parity slip shows up as a result that differs between repetitions or
from torch.  Results must be bitwise identical across repetitions (the kernels
use no floating-point atomics) and match torch to round-off.
"""

import numpy as np
import pytest
import torch

from paper_2305_19013_b200 import _lib
from paper_2305_19013_b200.problems import make_config

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)
REPS = 25


def _gram(Xs, Y, m, st):
    n, d = Y.shape[0], len(Xs)
    tab = torch.tensor([x.data_ptr() for x in Xs], dtype=torch.int64, device=DEV)
    chunks = _lib.query("ekcg_gram_chunks", n, d, m, m)
    part = torch.empty(chunks * d * m * m, dtype=torch.float64, device=DEV)
    G = torch.empty(d * m * m, dtype=torch.float64, device=DEV)
    _lib.call("ekcg_gram", tab.data_ptr(), m, d, m, Y.data_ptr(), m, m, n, part.data_ptr(), None, st)
    _lib.call("ekcg_reduce", part.data_ptr(), chunks, d * m * m, G.data_ptr(), None, st)
    return G


def _update(Qs, C, W, m, st):
    tab = torch.tensor([q.data_ptr() for q in Qs], dtype=torch.int64, device=DEV)
    out = torch.empty_like(W)
    _lib.call("ekcg_block_update", tab.data_ptr(), m, len(Qs), m, C.data_ptr(), W.data_ptr(), m, out.data_ptr(), m,
              m, 1.0, -1.0, W.shape[0], None, st)
    return out


def _case(kind):
    """(launch(st) -> tensor, torch reference, rel tol)."""
    g = torch.Generator(device=DEV).manual_seed(7)
    rnd = lambda *s: torch.randn(*s, dtype=torch.float64, device=DEV, generator=g)  # noqa: E731
    if kind in ("gram16_d1", "gram16_d5", "gram32_d3"):
        m, d = (16, 1) if kind == "gram16_d1" else (16, 5) if kind == "gram16_d5" else (32, 3)
        n = 400_003
        Xs, Y = [rnd(n, m) for _ in range(d)], rnd(n, m)
        return (lambda st: _gram(Xs, Y, m, st)), torch.stack([x.T @ Y for x in Xs]).reshape(-1), 1e-12
    if kind in ("update16_d7", "update32_d3"):
        m, d = (16, 7) if kind == "update16_d7" else (32, 3)
        n = 400_003
        Qs, W, C = [rnd(n, m) for _ in range(d)], rnd(n, m), rnd(d * m, m) * 0.1
        ref = W - sum(Qs[i] @ C[i * m:(i + 1) * m] for i in range(d))
        return (lambda st: _update(Qs, C, W, m, st)), ref, 1e-12
    idx, edge, m = {"march3d": (3, 64, 32), "march2d": (5, 1024, 64), "march3d_m16": (2, 64, 16)}[kind]
    prob = make_config(idx, edge)
    op = prob.stencil(DEV)
    A = prob.csr()
    X = rnd(prob.n, m)
    rows = torch.from_numpy(np.repeat(np.arange(prob.n), np.diff(A.row_ptr))).to(DEV)
    cols, vals = torch.from_numpy(A.col_idx).to(DEV), torch.from_numpy(A.values).to(DEV)
    ref = torch.zeros_like(X).index_add_(0, rows, vals[:, None] * X[cols])

    def run(st):
        Y = torch.empty_like(X)
        assert _lib.query("ekcg_spmm_stencil_kernel", 1, op.desc_ref(), X.data_ptr(), m, Y.data_ptr(), m, m, None,
                          st) == 0
        return Y
    return run, ref, 1e-13


@pytest.mark.parametrize("kind", ["gram16_d1", "gram16_d5", "gram32_d3", "update16_d7", "update32_d3", "march3d",
                                  "march2d", "march3d_m16"])
def test_ring_kernel_bitwise_under_contention(kind):
    run, ref, tol = _case(kind)
    main = torch.cuda.current_stream()
    noise = torch.cuda.Stream()
    a = torch.randn(1536, 1536, dtype=torch.float64, device=DEV)
    first = run(main.cuda_stream).clone()
    torch.cuda.synchronize()
    err = (first - ref).abs().max().item() / ref.abs().max().item()
    assert err <= tol, err
    for rep in range(REPS):
        noise.wait_stream(main)
        with torch.cuda.stream(noise):
            for _ in range(rep % 4):  # 0..3 GEMMs in flight beside the ring kernel
                a = a @ a * (1.0 / 1536.0)
        out = run(main.cuda_stream)
        assert torch.equal(out, first), (kind, rep)
    torch.cuda.synchronize()
