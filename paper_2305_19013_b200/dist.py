"""Row sharding across GPUs: slabs of whole grid layers, neighbour
halo exchange and small allreduces, over torch.distributed (NCCL on GPUs, gloo
on CPU for the host-side tests).

Rows are kept in the reference's x-fastest order; rank p owns the contiguous
rows of layers [l0, l1) of the slowest grid axis (z in 3-D, y in 2-D).  The
T^t split is row-local (a rank may own rows of several subdomains), the
stencil SpMM needs one layer of halo from each neighbour, and every Gram /
norm is a sum of per-rank partials reduced with one allreduce.  NCCL hands
every rank the same reduced bytes, so the m x m factorizations computed
redundantly on each rank agree bit for bit.
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
        """Fill the halo layers of an extended row block.

        `ext` is a flat tensor of shard.ext_rows * ld values laid out as
        [lower halo | local rows | upper halo]; the first local layer goes to
        the lower neighbour's upper halo and the last local layer to the upper
        neighbour's lower halo.
        """
        if self.world == 1:
            return
        h = shard.halo * ld
        nl = shard.n_local * ld
        ops = []
        if shard.has_lo:
            ops.append(dist.P2POp(dist.isend, ext[h:2 * h], shard.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, ext[0:h], shard.rank - 1, self.group))
        if shard.has_hi:
            ops.append(dist.P2POp(dist.isend, ext[nl:nl + h], shard.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, ext[nl + h:nl + 2 * h], shard.rank + 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

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
        """Fill the halo rows of an extended block [lo | local | hi] of a CsrShard:
        pack the rows each peer needs (send_idx[q]: device index tensors of local
        rows) and receive each peer's rows straight into their halo range."""
        if self.world == 1:
            return
        E = ext[: shard.ext_rows * ld].view(shard.ext_rows, ld)
        loc = E[shard.lo:shard.lo + shard.n_local]
        ops, keep = [], []
        for q, idx in send_idx.items():
            buf = loc.index_select(0, idx).contiguous()
            keep.append(buf)
            ops.append(dist.P2POp(dist.isend, buf.view(-1), q, self.group))
        for q, (start, count, _) in shard.recv.items():
            ops.append(dist.P2POp(dist.irecv, E[start:start + count].view(-1), q, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

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
