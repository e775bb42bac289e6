"""Multi-rank host logic of the row-sharded engine, on CPU with gloo (world 2 and 3).

Checks the slab decomposition, the halo exchange, the partial-sum allreduce
and the row gather -- and that a stencil product assembled from per-rank
slabs plus exchanged halos equals the global product (the data flow the
sharded GPU engine uses around its kernels).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ekcg_oracle as orc
from paper_2305_19013_b200.dist import Comm, CsrShard, RowShard, permute_csr, row_bounds, subdomain_order
from paper_2305_19013_b200.problems import box_owner, diffusion_csr


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, shape, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = Comm()
        sh = RowShard(shape, rank, world)
        n = int(np.prod(shape))
        rng = np.random.default_rng(7)
        X = rng.standard_normal((n, m))
        kappa = np.exp(rng.uniform(-2, 2, n))
        A = diffusion_csr(shape, kappa)
        # extended local block: [halo | local | halo], halos filled by the exchange
        ext = torch.zeros(sh.ext_rows * m, dtype=torch.float64)
        loc = torch.from_numpy(X[sh.row_begin:sh.row_end].copy()).reshape(-1)
        ext[sh.halo * m:(sh.halo + sh.n_local) * m] = loc
        comm.halo_exchange(ext, m, sh)
        E = ext.reshape(sh.ext_rows, m).numpy()
        lo = sh.row_begin - sh.halo
        ok_halo = True
        if sh.has_lo:
            ok_halo &= np.array_equal(E[:sh.halo], X[lo:sh.row_begin])
        if sh.has_hi:
            ok_halo &= np.array_equal(E[sh.halo + sh.n_local:], X[sh.row_end:sh.row_end + sh.halo])
        # local rows of A X from the extended block only
        Y_loc = np.zeros((sh.n_local, m))
        for i in range(sh.row_begin, sh.row_end):
            for j in range(A.row_ptr[i], A.row_ptr[i + 1]):
                c = A.col_idx[j]
                assert lo <= c < sh.row_end + sh.halo
                Y_loc[i - sh.row_begin] += A.values[j] * E[c - lo]
        Y_ref = (A.to_dense() @ X)[sh.row_begin:sh.row_end]
        ok_prod = np.allclose(Y_loc, Y_ref, rtol=1e-13, atol=1e-12)
        # Gram partials -> allreduce equals the global Gram
        G = torch.from_numpy(X[sh.row_begin:sh.row_end].T @ Y_ref)
        comm.allreduce_(G)
        ok_gram = np.allclose(G.numpy(), X.T @ (A.to_dense() @ X), rtol=1e-12)
        # gather of uneven slabs
        full = comm.gather_rows(torch.from_numpy(X[sh.row_begin:sh.row_end, 0].copy()), sh)
        ok_gather = np.array_equal(full.numpy(), X[:, 0])
        q.put((rank, bool(ok_halo), bool(ok_prod), bool(ok_gram), bool(ok_gather)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape", [(2, (5, 4, 6)), (3, (4, 3, 7)), (2, (6, 9))])
def test_sharded_dataflow_gloo(world, shape):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, 3, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    results = sorted(q.get() for _ in range(world))
    for rank, ok_halo, ok_prod, ok_gram, ok_gather in results:
        assert ok_halo and ok_prod and ok_gram and ok_gather, (rank, ok_halo, ok_prod, ok_gram, ok_gather)


@pytest.mark.parametrize("layers,world", [(64, 1), (64, 2), (64, 8), (7, 3), (256, 8), (8192, 8)])
def test_row_shard_covers_rows(layers, world):
    shape = (4, 3, layers)
    shards = [RowShard(shape, r, world) for r in range(world)]
    assert shards[0].row_begin == 0 and shards[-1].row_end == 4 * 3 * layers
    for a, b in zip(shards, shards[1:]):
        assert a.row_end == b.row_begin
    sizes = [s.n_local // s.plane for s in shards]
    assert max(sizes) - min(sizes) <= 1
    assert not shards[0].has_lo and not shards[-1].has_hi
    with pytest.raises(ValueError):
        RowShard((4, 4), 0, 5)


def _random_spd_csr(n, rng):
    """Symmetric sparsity with far-off columns (non-banded) and a dominant diagonal."""
    rows, cols = [], []
    for i in range(n):
        k = rng.integers(1, 6)
        js = rng.choice(n, k, replace=False)
        for j in js:
            if j != i:
                rows += [i, j]
                cols += [j, i]
    M = np.zeros((n, n))
    M[rows, cols] = rng.uniform(-1, 0, len(rows))
    M = 0.5 * (M + M.T)
    M[np.arange(n), np.arange(n)] = np.abs(M).sum(axis=1) + 1.0
    rp = np.concatenate(([0], np.cumsum((M != 0).sum(axis=1)))).astype(np.int64)
    ci = np.nonzero(M)[1].astype(np.int64)
    return rp, ci, M[M != 0]


def _csr_worker(rank, world, port, kind, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = Comm()
        rng = np.random.default_rng(11)
        bounds = None
        if kind in ("grid", "subdomain"):
            A = diffusion_csr((8, 4, 6), np.exp(rng.uniform(-2, 2, 192)))
            rp, ci, vals = A.row_ptr, A.col_idx, A.values
        else:
            rp, ci, vals = _random_spd_csr(90, rng)
        n = len(rp) - 1
        X = rng.standard_normal((n, m))
        if kind == "subdomain":  # 4 x 2 x 2 boxes, whole subdomains per rank, interior rows first
            owner = box_owner((8, 4, 6), (4, 2, 2))
            order, bounds = subdomain_order(owner, 16, world, rp, ci)
            rp0, ci0, vals0 = rp, ci, vals
            rp, ci, vals = permute_csr(rp, ci, vals, order)
            # P A P^T keeps every row's products: the permuted product is the original's rows, bitwise
            assert np.array_equal(orc.csr_spmm(rp, ci, vals, X[order]), orc.csr_spmm(rp0, ci0, vals0, X)[order])
            X = X[order]
            per = 16 // world
            sub = owner[order]
            assert all(set(sub[bounds[p]:bounds[p + 1]] // per) == {p} for p in range(world))
        sh = CsrShard(rp, ci, rank, world, bounds=bounds).plan(comm)
        ext = torch.zeros(sh.ext_rows * m, dtype=torch.float64)
        ext.view(sh.ext_rows, m)[sh.lo:sh.lo + sh.n_local] = torch.from_numpy(X[sh.row_begin:sh.row_end])
        comm.csr_exchange(ext, m, sh, {q_: torch.from_numpy(v) for q_, v in sh.send.items()})
        E = ext.view(sh.ext_rows, m).numpy()
        halo_ok = (np.array_equal(E[:sh.lo], X[sh.lo_rows]) and
                   np.array_equal(E[sh.lo + sh.n_local:], X[sh.hi_rows]))
        e0, e1 = rp[sh.row_begin], rp[sh.row_end]
        lci = sh.local_col_idx.astype(np.int64)
        Y_loc = np.add.reduceat(vals[e0:e1][:, None] * E[lci], sh.local_row_ptr[:-1], axis=0)  # linalg.py:150
        Y_ref = orc.csr_spmm(rp, ci, vals, X)[sh.row_begin:sh.row_end]
        prod_ok = np.array_equal(Y_loc.view(np.int64), Y_ref.view(np.int64))  # same association: bitwise
        # interior rows reference no halo row (they run while the exchange is in flight)
        interior, boundary = sh.row_ranges()
        if interior is not None:
            a, b = interior
            seg = lci[sh.local_row_ptr[a]:sh.local_row_ptr[b]]
            prod_ok &= bool(np.all((seg >= sh.lo) & (seg < sh.lo + sh.n_local)))
            covered = sorted([interior] + boundary)
            prod_ok &= covered[0][0] == 0 and covered[-1][1] == sh.n_local and all(
                x[1] == y[0] for x, y in zip(covered, covered[1:]))
            if kind == "subdomain":
                prod_ok &= a == 0 and b > 0  # interior-first numbering
        full = comm.gather_rows(torch.from_numpy(X[sh.row_begin:sh.row_end, 0].copy()), sh)
        gather_ok = np.array_equal(full.numpy(), X[:, 0])
        q.put((rank, bool(halo_ok), bool(prod_ok), bool(gather_ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "grid"), (3, "grid"), (2, "random"), (3, "random"),
                                        (2, "subdomain"), (4, "subdomain")])
def test_csr_sharded_dataflow_gloo(world, kind):
    """CSR row shards: the halo plan (requests exchanged once), the per-product exchange
    and a local product on [lo halo | local | hi halo] that equals the global rows bitwise."""
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_csr_worker, args=(r, world, port, kind, 4, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for rank, halo_ok, prod_ok, gather_ok in sorted(q.get() for _ in range(world)):
        assert halo_ok and prod_ok and gather_ok, (rank, halo_ok, prod_ok, gather_ok)


def test_csr_shard_single_rank_and_bounds():
    rp, ci, vals = _random_spd_csr(40, np.random.default_rng(2))
    sh = CsrShard(rp, ci, 0, 1)
    assert sh.lo == 0 and sh.ext_rows == 40 and not sh.recv
    assert np.array_equal(sh.local_col_idx, ci) and np.array_equal(sh.local_row_ptr, rp)
    b = row_bounds(10, 3)
    assert list(b) == [0, 4, 7, 10]
    with pytest.raises(ValueError):
        row_bounds(2, 3)


def test_stencil_row_ranges_cover_the_slab():
    for world in (1, 2, 4):
        for r in range(world):
            sh = RowShard((6, 5, 16), r, world)
            interior, boundary = sh.row_ranges()
            rngs = sorted(([interior] if interior else []) + boundary)
            assert rngs[0][0] == sh.row_begin and rngs[-1][1] == sh.row_end
            assert all(x[1] == y[0] for x, y in zip(rngs, rngs[1:]))
            if interior:  # the interior's stencil neighbours stay inside the slab
                assert interior[0] - sh.plane >= sh.row_begin or not sh.has_lo
                assert interior[1] + sh.plane <= sh.row_end or not sh.has_hi


def test_subdomain_order_needs_divisible_t():
    assert subdomain_order(np.zeros(10, dtype=np.int64), 3, 2) is None
    order, bounds = subdomain_order(np.repeat(np.arange(4), 5)[::-1].copy(), 4, 2)
    assert list(bounds) == [0, 10, 10 + 10] and sorted(order) == list(range(20))
