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

    def local_slice(self):
        return slice(self.row_begin, self.row_end)

    def __repr__(self):
        return f"RowShard(rank={self.rank}/{self.world}, rows=[{self.row_begin}, {self.row_end}), halo={self.halo})"


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
        out = []
        for r, p in enumerate(parts):
            s = RowShard(shard.shape, r, self.world)
            out.append(p[: s.n_local])
        return torch.cat(out)
