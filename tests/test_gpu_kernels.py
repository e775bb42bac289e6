"""Kernel-level parity on the GPU, through the C ABI (paper_2305_19013_b200._lib).

Integer/copy work (split) and the sparse products are bit-exact against the
reference's outputs; fp64 Gram/update/factorization kernels are compared with
a torch fp64 / numpy reference at the stated tolerances.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2305_19013_b200 as pk
from paper_2305_19013_b200 import _lib
from paper_2305_19013_b200.problems import make_config
from oracle import ekcg_oracle as orc

DEV = "cuda"


def dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a)).to(DEV, dtype)


def stream():
    return torch.cuda.current_stream().cuda_stream


def test_split_bitwise(kernels_golden):
    g = kernels_golden
    p = pk.Partition.from_owner(g["split_owner"], 3)
    W = p.split(g["split_v"])
    assert np.array_equal(W, g["split_W"])
    rng = np.random.default_rng(3)
    owner = rng.integers(0, 16, 100_003)
    owner[:16] = np.arange(16)
    v = rng.standard_normal(owner.size)
    v[::7] = -0.0
    q = pk.Partition.from_owner(owner, 16)
    Wd = q.split(v)
    ref = orc.split_block(owner, 16, v)
    assert np.array_equal(Wd.view(np.int64), ref.view(np.int64))  # bitwise incl. signed zeros


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_csr_spmm_bitwise(kernels_golden, tag):
    g = kernels_golden
    A = pk.SparseSpdMatrix(len(g[f"spmm_{tag}_rp"]) - 1, g[f"spmm_{tag}_rp"], g[f"spmm_{tag}_ci"],
                           g[f"spmm_{tag}_v"])
    X = g[f"spmm_{tag}_X"]
    assert np.array_equal(pk.spmm(A, X), g[f"spmm_{tag}_Y"])
    assert np.array_equal(pk.spmv(A, X[:, 3].copy()), g[f"spmv_{tag}_y"])
    for m in (1, 3, 8, 16, 64):
        assert np.array_equal(pk.spmm(A, X[:, :m].copy()), g[f"spmm_{tag}_Y"][:, :m])


@pytest.mark.parametrize("m", [1, 2, 4, 6, 12, 32, 64])
def test_csr_vectorized_equals_scalar_kernel(m):
    """Every CSR kernel form (ekcg_spmm_csr_kernel: 4 / 2 columns per thread, one thread
    per (row, column), the automatic choice) bitwise, on rows of 1..20 entries (the < 8
    fast path, the 8 / 9 boundary and the pairwise tail)."""
    rng = np.random.default_rng(m)
    n = 5000
    lens = rng.integers(1, 21, n)
    lens[:25] = np.arange(1, 26) % 21 + 1
    rp = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int32)
    vals = rng.standard_normal(rp[-1])
    X = dev(rng.standard_normal((n, m)))
    rp_d, ci_d, v_d = dev(rp, torch.int64), dev(ci, torch.int32), dev(vals)
    outs = []
    for form in (3, 4, 5, 0):
        Y = torch.full_like(X, float("nan"))
        rc = _lib.query("ekcg_spmm_csr_kernel", form, rp_d.data_ptr(), ci_d.data_ptr(), v_d.data_ptr(), X.data_ptr(),
                        m, Y.data_ptr(), m, n, m, None, stream())
        if rc != 0:  # the form does not apply to this width
            assert (form == 3 and m % 4) or (form == 4 and m % 2), (form, m, rc)
            continue
        outs.append(Y.cpu().numpy())
    for o in outs[1:]:
        assert np.array_equal(o.view(np.int64), outs[0].view(np.int64))
    ref = orc.csr_spmm(rp, ci.astype(np.int64), vals, X.cpu().numpy())
    assert np.array_equal(outs[0].view(np.int64), ref.view(np.int64))


@pytest.mark.parametrize("m", [16, 32, 64, 128])
def test_csr_pipelined_equals_vectorized(m):
    """The software-pipelined CSR kernel (256-bit and 128-bit accesses) against the
    vectorized one, bitwise, with enough rows that every thread walks several rows (the
    pipelined pairs / row pointers), rows of 1..20 entries and a ragged last warp."""
    rng = np.random.default_rng(100 + m)
    n = 300_001 if m <= 32 else 100_003
    lens = rng.integers(1, 21, n)
    lens[rng.random(n) < 0.7] = 7
    rp = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    ci = rng.integers(0, n, rp[-1]).astype(np.int32)
    vals = rng.standard_normal(rp[-1])
    X = dev(rng.standard_normal((n, m)))
    rp_d, ci_d, v_d = dev(rp, torch.int64), dev(ci, torch.int32), dev(vals)
    outs = []
    for form in (1, 3, 2):  # pipelined with 256-bit / 128-bit accesses, vectorized
        Y = torch.full_like(X, float("nan"))
        assert _lib.query("ekcg_spmm_csr_kernel", form, rp_d.data_ptr(), ci_d.data_ptr(), v_d.data_ptr(),
                          X.data_ptr(), m, Y.data_ptr(), m, n, m, None, stream()) == 0
        outs.append(Y.cpu().numpy())
    assert np.array_equal(outs[0].view(np.int64), outs[1].view(np.int64))
    assert np.array_equal(outs[2].view(np.int64), outs[1].view(np.int64))


@pytest.mark.parametrize("shift", [0, 2, 1])
def test_csr_offset_blocks(shift):
    """X and Y blocks starting `shift` doubles into their buffers (32-B aligned, 16-B only, 8-B only): the
    dispatch falls back from the 256-bit to the 128-bit to the scalar kernel, all bitwise equal to the oracle."""
    rng = np.random.default_rng(7 + shift)
    n, m = 20_011, 16
    lens = rng.integers(1, 12, n)
    rp = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    ci = rng.integers(0, n, rp[-1]).astype(np.int32)
    vals = rng.standard_normal(rp[-1])
    Xh = rng.standard_normal((n, m))
    Xbuf = torch.zeros(n * m + 8, dtype=torch.float64, device="cuda")
    Xbuf[shift:shift + n * m] = dev(Xh).reshape(-1)
    Ybuf = torch.full((n * m + 8,), float("nan"), dtype=torch.float64, device="cuda")
    rp_d, ci_d, v_d = dev(rp, torch.int64), dev(ci, torch.int32), dev(vals)
    _lib.call("ekcg_spmm_csr", rp_d.data_ptr(), ci_d.data_ptr(), v_d.data_ptr(), Xbuf.data_ptr() + 8 * shift, m,
              Ybuf.data_ptr() + 8 * shift, m, n, m, None, stream())
    Y = Ybuf[shift:shift + n * m].reshape(n, m).cpu().numpy()
    ref = orc.csr_spmm(rp, ci.astype(np.int64), vals, Xh)
    assert np.array_equal(Y.view(np.int64), ref.view(np.int64))


@pytest.mark.parametrize("idx,edge", [(1, 20), (2, 8), (3, 16), (4, 8), (5, 64)])
@pytest.mark.parametrize("m", [1, 2, 7, 16, 32])
def test_stencil_equals_csr_bitwise(idx, edge, m):
    prob = make_config(idx, edge)
    A = prob.csr()
    op = prob.stencil()
    X = np.random.default_rng(idx * 100 + m).standard_normal((prob.n, m))
    X[::5, 0] = 0.0
    Xd = dev(X)
    Yd = torch.empty_like(Xd)
    op.apply(Xd, m, Yd, m, m)
    ref = orc.csr_spmm(A.row_ptr, A.col_idx, A.values, X)
    assert np.array_equal(Yd.cpu().numpy(), ref)
    assert np.array_equal(pk.spmm(A, X), ref)


@pytest.mark.parametrize("idx,edge", [(3, 32), (3, 40), (5, 128), (5, 96)])
@pytest.mark.parametrize("m", [16, 32, 64])
def test_march_tile_field_bitwise(idx, edge, m):
    """Plane march on the config-3 / config-5 tile fields (per-tile coefficient fast
    path for tile-interior nodes, face lookups elsewhere) against the reference
    association on the assembled CSR, bitwise."""
    prob = make_config(idx, edge, device_rhs=False)
    A = prob.csr()
    op = prob.stencil()
    X = np.random.default_rng(idx + edge + m).standard_normal((prob.n, m))
    Xd = dev(X)
    Yd = torch.empty_like(Xd)
    assert _lib.query("ekcg_spmm_stencil_kernel", 1, op.desc_ref(), Xd.data_ptr(), m, Yd.data_ptr(), m, m, None,
                      stream()) == 0  # the plane march at any size
    ref = orc.csr_spmm(A.row_ptr, A.col_idx, A.values, X)
    assert np.array_equal(Yd.cpu().numpy().view(np.int64), ref.view(np.int64))


@pytest.mark.parametrize("shape,kappa", [((17, 5, 9), None), ((67, 3), None), ((33, 33, 3), "tile"),
                                         ((2, 2, 2), None), ((130, 7), "node"), ((21, 19, 11), "node")])
@pytest.mark.parametrize("m", [4, 12, 16, 20, 64])
def test_stencil_march_kernel(shape, kappa, m):
    """Plane-marching kernel (form 1) vs the row kernel (form 2) vs the CSR oracle,
    on ragged tiles, partial column chunks and plane-aligned row ranges."""
    import ctypes
    rng = np.random.default_rng(len(shape) * 1000 + m + shape[0])
    n = int(np.prod(shape))
    if kappa == "tile":
        tile = (4,) * len(shape)
        need = tuple(-(-s // 4) for s in shape)[::-1]
        op = pk.StencilOperator(shape, 10.0 ** rng.uniform(-2, 2, need), tile=tile)
    elif kappa == "node":
        op = pk.StencilOperator(shape, 10.0 ** rng.uniform(-3, 3, n))
    else:
        op = pk.StencilOperator(shape, 2.5)
    A = op.to_csr()
    X = rng.standard_normal((n, m))
    X[::3, 1] = 0.0
    ref = orc.csr_spmm(A.row_ptr, A.col_idx, A.values, X)
    Xd = dev(X)
    outs = []
    for form in (1, 2):  # plane march at any size, row-parallel kernel
        Yd = torch.full_like(Xd, np.nan)
        rc = _lib.query("ekcg_spmm_stencil_kernel", form, op.desc_ref(), Xd.data_ptr(), m, Yd.data_ptr(), m, m,
                        None, stream())
        assert rc == 0 or (form == 1 and m % 4), (form, m, rc)
        outs.append(Yd.cpu().numpy() if rc == 0 else ref)
    # plane-aligned row range (one shard's slab), march when it applies
    plane = n // shape[-1]
    lo, hi = plane * (shape[-1] // 3), plane * max(shape[-1] // 3 + 1, (2 * shape[-1]) // 3)
    d = op._desc
    sub = type(d)()
    ctypes.pointer(sub)[0] = d
    sub.row_begin, sub.row_end = lo, hi
    Yd = torch.full_like(Xd, np.nan)
    if _lib.query("ekcg_spmm_stencil_kernel", 1, ctypes.byref(sub), Xd.data_ptr(), m, Yd.data_ptr(), m, m, None,
                  stream()) != 0:
        _lib.call("ekcg_spmm_stencil", ctypes.byref(sub), Xd.data_ptr(), m, Yd.data_ptr(), m, m, None, stream())
    part = Yd.cpu().numpy()
    assert np.array_equal(outs[0], ref)
    assert np.array_equal(outs[1], ref)
    assert np.array_equal(part[lo:hi], ref[lo:hi])
    assert np.isnan(part[:lo]).all() and np.isnan(part[hi:]).all()


def test_spmm_strided_slabs():
    prob = make_config(2, 8)
    op = prob.stencil()
    A = prob.csr()
    n, t, s = prob.n, 4, 3
    V = torch.zeros((n, s * t), dtype=torch.float64, device=DEV)
    V[:, :t] = dev(np.random.default_rng(1).standard_normal((n, t)))
    for i in range(1, s):
        op.apply(V.data_ptr() + 8 * (i - 1) * t, s * t, V.data_ptr() + 8 * i * t, s * t, t)
    Vh = V.cpu().numpy()
    ref = Vh[:, :t]
    for i in range(1, s):
        ref = orc.csr_spmm(A.row_ptr, A.col_idx, A.values, ref)
        assert np.array_equal(Vh[:, i * t:(i + 1) * t], ref)


@pytest.mark.parametrize("m1,m2", [(1, 1), (3, 1), (5, 7), (8, 8), (16, 16), (32, 32), (64, 64), (16, 1),
                                   (20, 20), (64, 32)])
@pytest.mark.parametrize("n", [1, 37, 4099, 200_000])
def test_gram_multi_block(m1, m2, n):
    rng = np.random.default_rng(m1 * 1000 + m2 + n)
    d = 3
    Xs = [dev(rng.standard_normal((n, m1))) for _ in range(d)]
    Y = dev(rng.standard_normal((n, m2)))
    tab = torch.tensor([x.data_ptr() for x in Xs], dtype=torch.int64, device=DEV)
    chunks = _lib.query("ekcg_gram_chunks", n, d, m1, m2)
    part = torch.empty(chunks * d * m1 * m2, dtype=torch.float64, device=DEV)
    out = torch.empty(d * m1 * m2, dtype=torch.float64, device=DEV)
    _lib.call("ekcg_gram", tab.data_ptr(), m1, d, m1, Y.data_ptr(), m2, m2, n, part.data_ptr(), None, stream())
    _lib.call("ekcg_reduce", part.data_ptr(), chunks, d * m1 * m2, out.data_ptr(), None, stream())
    got = out.view(d, m1, m2)
    for i in range(d):
        ref = Xs[i].T @ Y
        scale = (Xs[i].abs().T @ Y.abs()).max().item() + 1e-300
        assert (got[i] - ref).abs().max().item() <= 1e-13 * scale


@pytest.mark.parametrize("m", [4, 8, 16, 32, 64])
def test_vec256_paths_bitwise(m):
    """X^T y (m2 = 1) and the fused x / r update with 256-bit row loads (32-B aligned blocks) against
    the 128-bit loads (the same blocks 16 B off a 32-B boundary): the same products and sums, so bitwise
    equal; plus a tolerance check on X^T y."""
    rng = np.random.default_rng(240 + m)
    n, d = 300_007, 2
    host = [rng.standard_normal((n, m)) for _ in range(d)]
    y = dev(rng.standard_normal(n))
    chunks = _lib.query("ekcg_gram_chunks", n, d, m, 1)
    part = torch.empty(chunks * d * m, dtype=torch.float64, device=DEV)
    alpha = dev(rng.standard_normal(m) * 1e-2)
    vchunks = _lib.query("ekcg_vec_chunks", n)
    outs = {}
    for v, off in ((1, 0), (0, 2)):  # offset 2 doubles: 16-B aligned, not 32-B
        bufs = [torch.empty(n * m + 4, dtype=torch.float64, device=DEV) for _ in range(d)]
        Xs = [b[off:off + n * m].view(n, m) for b in bufs]
        for X, h in zip(Xs, host):
            X.copy_(torch.from_numpy(h))
        assert all((X.data_ptr() % 32 == 0) == (v == 1) for X in Xs)
        tab = torch.tensor([x.data_ptr() for x in Xs], dtype=torch.int64, device=DEV)
        g = torch.empty(d * m, dtype=torch.float64, device=DEV)
        _lib.call("ekcg_gram", tab.data_ptr(), m, d, m, y.data_ptr(), 1, 1, n, part.data_ptr(), None, stream())
        _lib.call("ekcg_reduce", part.data_ptr(), chunks, d * m, g.data_ptr(), None, stream())
        x, r = dev(rng.standard_normal(n) * 0 + 1.0), y.clone()
        vp = torch.empty(vchunks, dtype=torch.float64, device=DEV)
        _lib.call("ekcg_xr_update", Xs[0].data_ptr(), m, Xs[1].data_ptr(), m, alpha.data_ptr(), m, x.data_ptr(),
                  r.data_ptr(), n, vp.data_ptr(), None, stream())
        outs[v] = [t.cpu().numpy() for t in (g, x, r, vp)]
    for a, b in zip(outs[1], outs[0]):
        assert np.array_equal(a.view(np.int64), b.view(np.int64))
    ref = torch.stack([X.T @ y for X in Xs]).reshape(-1).cpu().numpy()
    assert np.max(np.abs(outs[1][0] - ref)) <= 1e-12 * np.max(np.abs(ref))

@pytest.mark.parametrize("n", [37, 4099, 200_000])
@pytest.mark.parametrize("m", [16, 32, 64])
def test_gram_self_symmetric_shortcut(n, m):
    """X^T X (the Pre-CholQR Gram): at m = 32 / 64 only the 8 x 8 tiles on and above the
    diagonal are formed and each is stored with its mirror, at m = 16 / 32 the block is
    streamed once and read as both operands; bitwise equal to X^T Y with Y a copy of X."""
    X = dev(np.random.default_rng(n).standard_normal((n, m)))
    Xc = X.clone()
    tab = torch.tensor([X.data_ptr()], dtype=torch.int64, device=DEV)
    chunks = _lib.query("ekcg_gram_chunks", n, 1, m, m)
    outs = []
    for Y in (X, Xc):
        part = torch.empty(chunks * m * m, dtype=torch.float64, device=DEV)
        G = torch.empty(m * m, dtype=torch.float64, device=DEV)
        _lib.call("ekcg_gram", tab.data_ptr(), m, 1, m, Y.data_ptr(), m, m, n, part.data_ptr(), None, stream())
        _lib.call("ekcg_reduce", part.data_ptr(), chunks, m * m, G.data_ptr(), None, stream())
        outs.append(G.view(m, m))
    assert torch.equal(outs[0], outs[1])
    assert torch.equal(outs[0], outs[0].T)
    assert (outs[0] - X.T @ X).abs().max().item() <= 1e-13 * (X.abs().T @ X.abs()).max().item()


@pytest.mark.parametrize("n", [200_000, 600_000, 1_000_003])
def test_streamed_gram_many_ctas_per_sm(n):
    """Regression: the TMA ring refills a slot only after a proxy fence orders the
    consumers' generic reads before the async write.  Without it, 3+ co-resident
    CTAs per SM (the one-block m = 16 Gram: 3 per SM, several waves at these
    chunk counts) read refilled slots and ~1 % of the rows went wrong."""
    m = 16
    X = torch.randn(n, m, dtype=torch.float64, device=DEV)
    tab = torch.tensor([X.data_ptr()], dtype=torch.int64, device=DEV)
    ref = X.T @ X
    chunks = _lib.query("ekcg_gram_chunks", n, 1, m, m)
    assert chunks > 2 * torch.cuda.get_device_properties(DEV).multi_processor_count
    for _ in range(3):
        part = torch.empty(chunks * m * m, dtype=torch.float64, device=DEV)
        G = torch.empty(m * m, dtype=torch.float64, device=DEV)
        _lib.call("ekcg_gram", tab.data_ptr(), m, 1, m, X.data_ptr(), m, m, n, part.data_ptr(), None, stream())
        _lib.call("ekcg_reduce", part.data_ptr(), chunks, m * m, G.data_ptr(), None, stream())
        assert (G.view(m, m) - ref).abs().max().item() <= 1e-13 * ref.abs().max().item()


def test_gram_deterministic():
    rng = np.random.default_rng(9)
    X = rng.standard_normal((300_001, 16))
    a = pk.gram(X, X)
    b = pk.gram(X, X)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("m1,m2", [(4, 4), (8, 8), (16, 16), (32, 32), (64, 64), (16, 8), (6, 6)])
@pytest.mark.parametrize("n", [5, 1000, 100_003])
@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_block_update(m1, m2, n, beta):
    rng = np.random.default_rng(n + m1 * 7 + m2)
    d = 4
    Qs = [dev(rng.standard_normal((n, m1))) for _ in range(d)]
    C = dev(rng.standard_normal((d * m1, m2)))
    Win = dev(rng.standard_normal((n, m2)))
    Wout = torch.empty_like(Win)
    tab = torch.tensor([q.data_ptr() for q in Qs], dtype=torch.int64, device=DEV)
    _lib.call("ekcg_block_update", tab.data_ptr(), m1, d, m1, C.data_ptr(), Win.data_ptr() if beta else None,
              m2, Wout.data_ptr(), m2, m2, beta, -1.0, n, None, stream())
    ref = beta * Win - sum(Qs[i] @ C[i * m1:(i + 1) * m1] for i in range(d))
    scale = sum((Qs[i].abs() @ C[i * m1:(i + 1) * m1].abs()) for i in range(d)).max().item() + 1.0
    assert (Wout - ref).abs().max().item() <= 1e-13 * scale
    # in place (Wout aliases Win), the CGS2 second pass
    if beta:
        W2 = Win.clone()
        _lib.call("ekcg_block_update", tab.data_ptr(), m1, d, m1, C.data_ptr(), W2.data_ptr(), m2, W2.data_ptr(),
                  m2, m2, 1.0, -1.0, n, None, stream())
        assert torch.equal(W2, Wout)


@pytest.mark.parametrize("m", [32, 64])
@pytest.mark.parametrize("d", [1, 2, 5, 7])
@pytest.mark.parametrize("n", [63, 70_001])
def test_wide_streamed_update_and_gram(m, d, n):
    """Wide-block kernels (m = 32 streamed, m = 64 smem-C / register-direct) against
    torch: every depth (C_i resident in smem or not), ragged last slab, in place."""
    rng = np.random.default_rng(m * 100 + d + n)
    Qs = [dev(rng.standard_normal((n, m))) for _ in range(d)]
    C = dev(rng.standard_normal((d * m, m)))
    Win = dev(rng.standard_normal((n, m)))
    tab = torch.tensor([q.data_ptr() for q in Qs], dtype=torch.int64, device=DEV)
    outs = []
    W = Win.clone()
    _lib.call("ekcg_block_update", tab.data_ptr(), m, d, m, C.data_ptr(), W.data_ptr(), m, W.data_ptr(),
              m, m, 1.0, -1.0, n, None, stream())
    chunks = _lib.query("ekcg_gram_chunks", n, d, m, m)
    part = torch.empty(chunks * d * m * m, dtype=torch.float64, device=DEV)
    G = torch.empty(d * m * m, dtype=torch.float64, device=DEV)
    _lib.call("ekcg_gram", tab.data_ptr(), m, d, m, Win.data_ptr(), m, m, n, part.data_ptr(), None, stream())
    _lib.call("ekcg_reduce", part.data_ptr(), chunks, d * m * m, G.data_ptr(), None, stream())
    outs.append((W, G.view(d, m, m)))
    ref = Win - sum(Qs[i] @ C[i * m:(i + 1) * m] for i in range(d))
    scale = sum((Qs[i].abs() @ C[i * m:(i + 1) * m].abs()) for i in range(d)).max().item() + 1.0
    for W, G in outs:
        assert (W - ref).abs().max().item() <= 1e-13 * scale
        for i in range(d):
            gref = Qs[i].T @ Win
            gscale = (Qs[i].abs().T @ Win.abs()).max().item() + 1e-300
            assert (G[i] - gref).abs().max().item() <= 1e-13 * gscale


@pytest.mark.parametrize("m", [3, 16, 32, 64])
@pytest.mark.parametrize("n", [1, 1001, 70_003])
def test_tri_apply(m, n):
    """ekcg_tri_apply (W S, S upper triangular) equals the full block update bitwise
    (the skipped blocks multiply exact zeros) and torch to 1e-13."""
    rng = np.random.default_rng(m + n)
    W = dev(rng.standard_normal((n, m)))
    S = dev(np.triu(rng.standard_normal((m, m))))
    tab = torch.tensor([W.data_ptr()], dtype=torch.int64, device=DEV)
    out_tri, out_full = torch.empty_like(W), torch.empty_like(W)
    _lib.call("ekcg_tri_apply", tab.data_ptr(), m, S.data_ptr(), out_tri.data_ptr(), m, m, n, None, stream())
    _lib.call("ekcg_block_update", tab.data_ptr(), m, 1, m, S.data_ptr(), None, m, out_full.data_ptr(), m, m,
              0.0, 1.0, n, None, stream())
    assert torch.equal(out_tri, out_full)
    scale = (W.abs() @ S.abs()).max().item() + 1.0
    assert (out_tri - W @ S).abs().max().item() <= 1e-13 * scale


@pytest.mark.parametrize("m", [1, 2, 6, 16, 64])
def test_cholesky_and_trsm(m):
    rng = np.random.default_rng(m)
    W = rng.standard_normal((3 * m + 5, m))
    B = W.T @ W
    R = pk.cholesky_small(B)
    ref = orc.small_cholesky(B)
    assert np.allclose(R, ref, rtol=1e-11, atol=1e-12 * np.abs(ref).max())
    assert np.allclose(R.T @ R, B, rtol=1e-12, atol=1e-12 * np.abs(B).max())
    X = rng.standard_normal((50, m))
    Y = pk.trsm_right_inv(X, R)
    assert np.allclose(Y @ R, X, rtol=1e-12, atol=1e-11)


def test_cholesky_known_answer_and_breakdown(kernels_golden):
    R = pk.cholesky_small(np.array([[4.0, 2.0], [2.0, 5.0]]))
    assert np.array_equal(R, np.array([[2.0, 1.0], [0.0, 2.0]]))
    with pytest.raises(pk.Breakdown, match="pivot .* at column 1"):
        pk.cholesky_small(np.array([[1.0, 1.0], [1.0, 1.0]]))


def test_norm_and_gram_api(kernels_golden):
    g = kernels_golden
    G = pk.gram(g["gram_X"], g["gram_Y"])
    assert np.allclose(G, g["gram_G"], rtol=1e-13, atol=1e-13)
    v = np.random.default_rng(0).standard_normal(12345)
    assert abs(pk.norm2(v) - np.linalg.norm(v)) <= 1e-14 * np.linalg.norm(v)


def test_launch_counter_moves():
    before = _lib.query("ekcg_launch_count")
    pk.norm2(np.ones(10))
    assert _lib.query("ekcg_launch_count") >= before + 2


def test_public_api_accepts_misaligned_views():
    """Caller tensors at odd element offsets (not 16-/32-B aligned) go through the
    public gram / trsm / norm wrappers (copied to aligned storage first) instead of
    faulting in the bulk-copy / 256-bit kernels."""
    rng = np.random.default_rng(5)
    n, m = 50_001, 16
    buf = dev(rng.standard_normal(n * m + 3))
    X = buf[1:1 + n * m].view(n, m)
    assert X.data_ptr() % 16 != 0
    G = pk.gram(X, X)
    ref = X.T @ X
    assert (G - ref).abs().max().item() <= 1e-12 * ref.abs().max().item()
    R = torch.linalg.cholesky(ref).T.contiguous()
    Y = pk.trsm_right_inv(X, R)
    assert (Y @ R - X).abs().max().item() <= 1e-10 * X.abs().max().item()
    assert abs(pk.norm2(buf[1:]) - torch.linalg.vector_norm(buf[1:]).item()) <= 1e-12 * pk.norm2(buf[1:])


def test_nan_residual_reports_maxiter():
    """A NaN residual stops the solve with status 'maxiter', like the reference loop
    (solvers.py:357: `nan > tol * rho0` is false; :417: `nan <= tol * rho0` is false too)."""
    ctrl = torch.zeros(_lib.query("ekcg_ctrl_bytes"), dtype=torch.uint8, device=DEV)
    hist = torch.zeros(8, dtype=torch.float64, device=DEV)
    rho2 = torch.tensor([4.0], dtype=torch.float64, device=DEV)
    _lib.call("ekcg_start", ctrl.data_ptr(), rho2.data_ptr(), 1e-8, hist.data_ptr(), stream())
    rho2.fill_(float("nan"))
    _lib.call("ekcg_finish", ctrl.data_ptr(), rho2.data_ptr(), 1, 100, 0, hist.data_ptr(), stream())
    raw = ctrl.cpu().numpy()
    ints = raw[:32].view(np.int32)
    assert ints[0] == 0 and ints[1] == 2  # live cleared, status maxiter
