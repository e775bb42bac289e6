"""Worker for tests/test_gpu_multirank.py: the sharded engine at world >= 2 on ONE GPU.

Launched by torchrun (RANK / WORLD_SIZE from the environment); every rank uses
cuda:0.  NCCL refuses two ranks on one device, so the collectives go through
`HostComm`, a TEST-ONLY Comm that stages each allreduce / halo exchange /
gather through host memory over gloo.  The engine, its kernels, the shard plans
and the interior / boundary split of every product are the production ones;
only the transport differs.  No rank's kernel ever waits on another rank's
kernel (each exchange completes on the host before the consumer is launched),
so sharing one GPU cannot deadlock.

    torchrun --nproc-per-node 2 tests/multirank_worker.py OUT_DIR CASE [CASE ...]

Each case writes OUT_DIR/<case>.npz on rank 0 (history, iterations, status, x).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2305_19013_b200.dist import Comm  # noqa: E402


class HostComm(Comm):
    """Test-only transport: every collective staged through host memory over gloo."""

    def allreduce_(self, t):
        if self.world > 1:
            h = t.detach().cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM)
            t.copy_(h)
        return t

    def max_(self, t):
        if self.world > 1:
            h = t.detach().cpu()
            dist.all_reduce(h, op=dist.ReduceOp.MAX)
            t.copy_(h)
        return t

    def _p2p(self, sends, recvs):
        """sends: [(peer, device tensor)], recvs: [(peer, device tensor view)] -- completes before returning."""
        reqs, bufs = [], []
        for q, src in sends:
            reqs.append(dist.isend(src.detach().cpu().contiguous(), q))
        for q, dst in recvs:
            h = torch.empty(dst.numel(), dtype=dst.dtype)
            bufs.append((dst, h))
            reqs.append(dist.irecv(h, q))
        for r in reqs:
            r.wait()
        for dst, h in bufs:
            dst.copy_(h.view_as(dst))

    def halo_exchange_start(self, ext, ld, shard):
        if self.world == 1:
            return None
        h, nl = shard.halo * ld, shard.n_local * ld
        sends, recvs = [], []
        if shard.has_lo:
            sends.append((shard.rank - 1, ext[h:2 * h]))
            recvs.append((shard.rank - 1, ext[0:h]))
        if shard.has_hi:
            sends.append((shard.rank + 1, ext[nl:nl + h]))
            recvs.append((shard.rank + 1, ext[nl + h:nl + 2 * h]))
        self._p2p(sends, recvs)
        return None

    def csr_exchange_start(self, ext, ld, shard, send_idx):
        if self.world == 1:
            return None
        E = ext[: shard.ext_rows * ld].view(shard.ext_rows, ld)
        loc = E[shard.lo:shard.lo + shard.n_local]
        sends = [(q, loc.index_select(0, idx).reshape(-1)) for q, idx in send_idx.items()]
        recvs = [(q, E[start:start + count].reshape(-1)) for q, (start, count, _) in shard.recv.items()]
        self._p2p(sends, recvs)
        return None

    def gather_rows(self, local, shard):
        if self.world == 1:
            return local
        counts = [shard.n_local_of(r) for r in range(self.world)]
        pad = torch.zeros(max(counts), dtype=local.dtype)
        pad[: shard.n_local] = local.cpu()
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(parts, pad)
        return torch.cat([p[:c] for p, c in zip(parts, counts)]).to(local.device)


def parse_case(name):
    """'<form>-cfg<idx>-<edge>-<scheme>[-kmax<K>]', e.g. stencil-cfg2-16-cached."""
    parts = name.split("-")
    form, idx, edge, scheme = parts[0], int(parts[1][3:]), int(parts[2]), parts[3]
    kmax = int(parts[4][4:]) if len(parts) > 4 else None
    return form, idx, edge, scheme, kmax


def build(name, device):
    import paper_2305_19013_b200 as pk
    from paper_2305_19013_b200.problems import make_config
    form, idx, edge, scheme, kmax = parse_case(name)
    prob = make_config(idx, edge, device_rhs=False)
    kw = dict(prob.solver_kwargs)
    if kmax is not None:
        kw["kmax"] = kmax
    cfg = pk.SolverConfig(**kw)
    op = prob.stencil(device) if form == "stencil" else prob.csr()
    return prob, cfg, op, scheme


def main():
    out = Path(sys.argv[1])
    cases = sys.argv[2:]
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    from paper_2305_19013_b200.sharded import ShardedEngine
    try:
        for name in cases:
            prob, cfg, op, scheme = build(name, dev)
            eng = ShardedEngine(op, prob.partition, cfg, comm=HostComm(), device=dev)
            eng.cache_aq = {"cached": True, "lean": False}[scheme]
            x, rep = eng.solve(prob.b, x_star=prob.x_star)
            if rank == 0:
                np.savez(out / f"{name}.npz", history=np.asarray(rep.residual_history), iterations=rep.iterations,
                         status=rep.status, x=np.asarray(x), peak=rep.peak_block_vectors,
                         true_residual=rep.true_residual, decomposition=eng.decomposition,
                         interior=np.asarray(eng.shard.row_ranges()[0] or (0, 0)), n_local=eng.shard.n_local)
            del eng, x
            torch.cuda.empty_cache()
    finally:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
