"""Row sharding across GPUs over torch.distributed (NCCL on GPUs,
gloo on CPU for the host-side tests): the decompositions, the halo plans, and
the collectives the sharded engine issues.

* Stencil operators (`RowShard`): rank p owns the contiguous rows of whole
  grid layers [l0, l1) of the slowest axis (z in 3-D, y in 2-D), in the
  reference's x-fastest order.  The stencil SpMM needs one layer of halo from
  each neighbour.  DESIGN.md section 7 gives the halo volumes against box
  decompositions; for config 5 (8 x 8 boxes) and at G = 2 for every config the
  slabs are exactly whole t-subdomains (partition.py:14-68).
* CSR matrices (`CsrShard`): rows renumbered subdomain-major
  (`subdomain_order`), so rank p owns whole subdomains [p t/G, (p+1) t/G) --
  the t-subdomain decomposition of north_star -- with each rank's interior
  rows (no off-rank column) first.  The halo is every off-rank row the local
  entries reference, exchanged with whichever peers own them.

The T^t split is row-local either way, every Gram / norm is a sum of per-rank
partials reduced with one allreduce, and NCCL hands every rank the same
reduced bytes, so the m x m factorizations computed redundantly on each rank
agree bit for bit.  Exchanges come in start / wait halves so the engine can
run the interior rows of a product while the halo is in flight.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


class RowShard:
    """Rows [row_begin, row_end) of a grid with `halo` rows (one layer) per side."""

    def __init__(self, shape, rank, world):
        shape = tuple(int(s) for s in shape)
        layers = shape[-1]
        plane = int(np.prod(shape[:-1]))
        if world < 1 or world > layers:
            raise ValueError(f"cannot split {layers} grid layers over {world} ranks")
        base, extra = divmod(layers, world)
        l0 = rank * base + min(rank, extra)
        l1 = l0 + base + (1 if rank < extra else 0)
        self.shape = shape
        self.rank, self.world = rank, world
        self.layers = (l0, l1)
        self.plane = plane
        self.halo = plane
        self.row_begin = l0 * plane
        self.row_end = l1 * plane
        self.n = int(np.prod(shape))
        self.n_local = self.row_end - self.row_begin
        self.has_lo = rank > 0
        self.has_hi = rank < world - 1

    def row_ranges(self):
        """(interior, boundary) global row ranges: the interior needs no halo row, so
        it can run while the halo is exchanged; the boundary layers run after."""
        lo = self.row_begin + (self.plane if self.has_lo else 0)
        hi = self.row_end - (self.plane if self.has_hi else 0)
        if hi <= lo:
            return None, [(self.row_begin, self.row_end)]
        bnd = [r for r in ((self.row_begin, lo), (hi, self.row_end)) if r[1] > r[0]]
        return (lo, hi), bnd

    @property
    def ext_rows(self):
        return self.n_local + 2 * self.halo

    @property
    def lo(self):
        """Halo rows stored before the local rows of an extended block."""
        return self.halo

    def n_local_of(self, rank):
        return RowShard(self.shape, rank, self.world).n_local

    def local_slice(self):
        return slice(self.row_begin, self.row_end)

    def __repr__(self):
        return f"RowShard(rank={self.rank}/{self.world}, rows=[{self.row_begin}, {self.row_end}), halo={self.halo})"


def subdomain_order(owner, t, world, row_ptr=None, col_idx=None):
    """Subdomain-major renumbering for a CSR shard (the t-subdomain decomposition).

    Returns (order, bounds): new row i is old row order[i]; rank p owns new rows
    [bounds[p], bounds[p+1]) = the whole subdomains [p t/G, (p+1) t/G).  Within a
    rank, rows whose columns all stay on the rank (interior) come first, so one
    contiguous range can run while the halo is in flight.  None when t % G != 0.
    The order inside each class is ascending, like the paper's METIS renumbering
    a symmetric permutation: the SpMM keeps every row's entries (and bits), only
    the Gram reductions change order.
    """
    owner = np.asarray(owner, dtype=np.int64)
    if world < 1 or t % world:
        return None
    per = t // world
    rank_of = owner // per
    order = np.argsort(rank_of, kind="stable")
    counts = np.bincount(rank_of, minlength=world)
    bounds = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    if row_ptr is not None:
        row_ptr = np.asarray(row_ptr, dtype=np.int64)
        col_rank = rank_of[np.asarray(col_idx, dtype=np.int64)]
        row_of = np.repeat(np.arange(len(owner)), np.diff(row_ptr))
        off = np.zeros(len(owner), dtype=bool)
        np.logical_or.at(off, row_of, col_rank != rank_of[row_of])
        # per rank: interior rows first, then boundary rows (both ascending)
        key = rank_of * 2 + off.astype(np.int64)
        order = np.argsort(key, kind="stable")
    return order, bounds


def permute_csr(row_ptr, col_idx, values, order):
    """P A P^T for new row i = old row order[i]; every row keeps its entries in
    their stored order (column ids renumbered), so each row's products and their
    association -- hence the SpMM bits -- are the reference's."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    n = len(row_ptr) - 1
    inv = np.empty(n, dtype=np.int64)
    inv[order] = np.arange(n)
    lens = np.diff(row_ptr)[order]
    new_ptr = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
    starts = row_ptr[:-1][order]
    idx = np.repeat(starts - new_ptr[:-1], lens) + np.arange(new_ptr[-1])
    return new_ptr, inv[np.asarray(col_idx, dtype=np.int64)[idx]], np.asarray(values, dtype=np.float64)[idx]


def row_bounds(n, world):
    """Contiguous, balanced row ranges: rank p owns [b[p], b[p+1])."""
    if world < 1 or world > n:
        raise ValueError(f"cannot split {n} rows over {world} ranks")
    base, extra = divmod(n, world)
    return np.array([p * base + min(p, extra) for p in range(world + 1)], dtype=np.int64)


class CsrShard:
    """Rows [row_begin, row_end) of a general CSR matrix plus its halo plan.

    The halo is every off-slab column the local rows reference: `lo_rows`
    (global ids < row_begin, ascending) and `hi_rows` (>= row_end, ascending),
    stored before / after the local rows of an extended block [lo | local |
    hi].  `local_col_idx` addresses that extended block; the entries keep
    their storage (ascending global column) order, so the SpMM association --
    and its bits -- are the reference's.  `recv[q]` is the (start, count)
    range of the extended block that rank q fills; `send[q]` the local row ids
    this rank sends to q (set up by `plan`, one all-to-all at construction).
    """

    def __init__(self, row_ptr, col_idx, rank, world, bounds=None):
        row_ptr = np.asarray(row_ptr, dtype=np.int64)
        col_idx = np.asarray(col_idx, dtype=np.int64)
        n = len(row_ptr) - 1
        self.bounds = row_bounds(n, world) if bounds is None else np.asarray(bounds, dtype=np.int64)
        self.rank, self.world, self.n = rank, world, n
        self.row_begin, self.row_end = int(self.bounds[rank]), int(self.bounds[rank + 1])
        self.n_local = self.row_end - self.row_begin
        e0, e1 = row_ptr[self.row_begin], row_ptr[self.row_end]
        cols = col_idx[e0:e1]
        self.lo_rows = np.unique(cols[cols < self.row_begin])
        self.hi_rows = np.unique(cols[cols >= self.row_end])
        self.halo_lo, self.halo_hi = len(self.lo_rows), len(self.hi_rows)
        local = np.where(cols < self.row_begin, np.searchsorted(self.lo_rows, cols),
                         np.where(cols < self.row_end, self.halo_lo + cols - self.row_begin,
                                  self.halo_lo + self.n_local + np.searchsorted(self.hi_rows, cols)))
        self.local_row_ptr = row_ptr[self.row_begin:self.row_end + 1] - e0
        self.local_col_idx = local.astype(np.int32)
        # the longest run of local rows that reference no halo row: it runs during the exchange
        off = (cols < self.row_begin) | (cols >= self.row_end)
        lens = np.diff(self.local_row_ptr)
        needs = np.zeros(self.n_local, dtype=bool)
        if off.any():
            needs[np.repeat(np.arange(self.n_local), lens)[off]] = True
        self.interior = _longest_false_run(needs)
        # rows needed from each owner: contiguous ranges of the extended block
        self.recv = {}
        for rows, base in ((self.lo_rows, 0), (self.hi_rows, self.halo_lo + self.n_local)):
            owners = np.searchsorted(self.bounds, rows, side="right") - 1
            for q in np.unique(owners):
                idx = np.nonzero(owners == q)[0]
                self.recv[int(q)] = (base + int(idx[0]), len(idx), rows[idx])
        self.send = {}

    @property
    def lo(self):
        return self.halo_lo

    @property
    def ext_rows(self):
        return self.halo_lo + self.n_local + self.halo_hi

    def row_ranges(self):
        """(interior, boundary) local row ranges (see RowShard.row_ranges)."""
        a, b = self.interior
        if b <= a:
            return None, [(0, self.n_local)]
        return (a, b), [r for r in ((0, a), (b, self.n_local)) if r[1] > r[0]]

    def n_local_of(self, rank):
        return int(self.bounds[rank + 1] - self.bounds[rank])

    def plan(self, comm):
        """Exchange the request lists once: send[q] = local rows rank q needs."""
        if comm.world == 1:
            return self
        reqs = [None] * comm.world
        for q, (_, _, rows) in self.recv.items():
            reqs[q] = rows
        got = comm.exchange_objects(reqs)
        self.send = {q: (np.asarray(r, dtype=np.int64) - self.row_begin) for q, r in enumerate(got)
                     if r is not None and len(r)}
        return self


def _longest_false_run(mask):
    """[a, b) of the longest run of False in a boolean vector ((0, 0) if none)."""
    if mask.size == 0:
        return 0, 0
    x = np.concatenate(([True], mask, [True]))
    edges = np.flatnonzero(np.diff(x.astype(np.int8)))  # run starts (True->False) and ends
    starts, ends = edges[0::2], edges[1::2]
    if starts.size == 0:
        return 0, 0
    j = int(np.argmax(ends - starts))
    return int(starts[j]), int(ends[j])


class Comm:
    """The collectives the sharded engine needs; single-process when world == 1."""

    def __init__(self, group=None):
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1

    def allreduce_(self, t):
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def max_(self, t):
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t

    def halo_exchange(self, ext, ld, shard):
        self.wait(self.halo_exchange_start(ext, ld, shard))

    @staticmethod
    def wait(works):
        """Make the current stream wait for a started exchange (NCCL: a stream wait, not a host block)."""
        for w in works or ():
            w.wait()

    def halo_exchange_start(self, ext, ld, shard):
        """Start filling the halo layers of an extended row block; returns the works.

        `ext` is a flat tensor of shard.ext_rows * ld values laid out as
        [lower halo | local rows | upper halo]; the first local layer goes to
        the lower neighbour's upper halo and the last local layer to the upper
        neighbour's lower halo.  The sends read only the first / last local
        layers and the receives write only the halos, so kernels on the current
        stream that read the local rows may run while the works are in flight.
        """
        if self.world == 1:
            return None
        h = shard.halo * ld
        nl = shard.n_local * ld
        ops = []
        if shard.has_lo:
            ops.append(dist.P2POp(dist.isend, ext[h:2 * h], shard.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, ext[0:h], shard.rank - 1, self.group))
        if shard.has_hi:
            ops.append(dist.P2POp(dist.isend, ext[nl:nl + h], shard.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, ext[nl + h:nl + 2 * h], shard.rank + 1, self.group))
        return dist.batch_isend_irecv(ops) if ops else None

    def exchange_objects(self, per_rank):
        """Send per_rank[q] to rank q; return the list received from every rank."""
        if self.world == 1:
            return [per_rank[0]]
        out = [None] * self.world
        gathered = [None] * self.world
        dist.all_gather_object(gathered, per_rank, group=self.group)
        for q in range(self.world):
            out[q] = gathered[q][self.rank]
        return out

    def csr_exchange(self, ext, ld, shard, send_idx):
        self.wait(self.csr_exchange_start(ext, ld, shard, send_idx))

    def csr_exchange_start(self, ext, ld, shard, send_idx):
        """Start filling the halo rows of an extended block [lo | local | hi] of a
        CsrShard: pack the rows each peer needs (send_idx[q]: device index tensors
        of local rows) and receive each peer's rows straight into their halo range."""
        if self.world == 1:
            return None
        E = ext[: shard.ext_rows * ld].view(shard.ext_rows, ld)
        loc = E[shard.lo:shard.lo + shard.n_local]
        ops, keep = [], []
        for q, idx in send_idx.items():
            buf = loc.index_select(0, idx).contiguous()
            keep.append(buf)
            ops.append(dist.P2POp(dist.isend, buf.view(-1), q, self.group))
        for q, (start, count, _) in shard.recv.items():
            ops.append(dist.P2POp(dist.irecv, E[start:start + count].view(-1), q, self.group))
        if not ops:
            return None
        works = dist.batch_isend_irecv(ops)
        self._keep = keep  # packed send buffers live until the next exchange is issued
        return works

    def gather_rows(self, local, shard):
        """Concatenate every rank's local rows (uneven slabs padded for all_gather)."""
        if self.world == 1:
            return local
        n_max = torch.tensor([shard.n_local], device=local.device, dtype=torch.int64)
        self.max_(n_max)
        n_max = int(n_max.item())
        pad = torch.zeros(n_max, dtype=local.dtype, device=local.device)
        pad[: shard.n_local] = local
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(parts, pad, group=self.group)
        return torch.cat([p[: shard.n_local_of(r)] for r, p in enumerate(parts)])
