"""Row-sharded multi-GPU engine: one process per GPU.

Each rank owns a slab of whole grid layers (dist.RowShard) and runs the same
kernel sequence as engine.DeviceEngine on its local rows:

* blocks that feed the stencil (the candidate / s-step chain block, W0, every
  retained W_k, x) are stored with one halo layer on each side and exchanged
  with the neighbours right before each operator application;
* every split-K reduction (CGS2 coefficients, Graw, G, alpha, |r|^2) is
  reduced locally, then summed across ranks with one NCCL allreduce, and the
  m x m factorizations / stop test run redundantly on every rank from
  identical bytes -- so all ranks take the same decisions;
* the stencil kernels address rows globally (EkcgStencil.row_begin/row_end),
  so the same sm_100a kernels serve one GPU and a shard.

General CSR matrices (the reference's SparseSpdMatrix) shard by balanced
contiguous row ranges (dist.CsrShard): each rank keeps the local rows with
column indices remapped into its extended block [lo halo | local | hi halo],
and before each product receives exactly the off-slab rows its entries
reference (one batched send/recv with every peer that owns some of them).

Scope: stencil and CSR operators, SRE-CG2 / SRE-CG with s >= 1, full / trunc /
restart retention; the cached-A Q scheme, or the lean one (no A Q cache, one
operator application per CGS2 pass) when the cached blocks do not fit.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .dist import Comm, CsrShard, RowShard, permute_csr, subdomain_order
from .partition import Partition
from .engine import F64, DeviceEngine, _Block
from .operators import CsrOperator, StencilOperator


class _LocalCsr:
    """The local rows of a CsrShard as a CSR whose columns index the extended block."""

    def __init__(self, row_ptr, values, shard):
        e0, e1 = int(row_ptr[shard.row_begin]), int(row_ptr[shard.row_end])
        self.n = shard.n_local
        self.row_ptr = shard.local_row_ptr
        self.col_idx = shard.local_col_idx
        self.values = np.ascontiguousarray(np.asarray(values)[e0:e1], dtype=np.float64)


class ShardedEngine(DeviceEngine):
    """decomposition: "subdomain" (CSR: rows renumbered subdomain-major, whole
    t-subdomains per rank, dist.subdomain_order; needs t % G == 0) or "rows"
    (balanced contiguous row ranges); stencil operators always shard by layers."""

    def __init__(self, op, partition, cfg, comm=None, device=None, decomposition="subdomain", overlap=True):
        if cfg.preconditioner is not None:
            raise ValueError("the sharded engine runs unpreconditioned")
        if cfg.method not in ("sre-cg2", "sre-cg") or cfg.switch_tol is not None:
            raise ValueError("the sharded engine runs SRE-CG2 / SRE-CG without the flexible switch")
        comm = comm if comm is not None else Comm()
        self.stencil = isinstance(op, StencilOperator)
        self.order = None  # new row i = global row order[i] (CSR subdomain decomposition)
        self.overlap = overlap  # run interior rows while the halo is exchanged
        if self.stencil:
            shard = RowShard(op.shape, comm.rank, comm.world)
            local_op = op
        else:
            host = op.host if isinstance(op, CsrOperator) else op
            if not all(hasattr(host, a) for a in ("n", "row_ptr", "col_idx", "values")):
                raise TypeError("the sharded engine needs a StencilOperator or a CSR matrix")
            rp, ci, vals = host.row_ptr, host.col_idx, host.values
            bounds = None
            plan = (subdomain_order(partition.owner(), partition.t, comm.world, rp, ci)
                    if decomposition == "subdomain" else None)
            if plan is not None:
                self.order, bounds = plan
                rp, ci, vals = permute_csr(rp, ci, vals, self.order)
                partition = Partition.from_owner(np.asarray(partition.owner())[self.order], partition.t)
            shard = CsrShard(rp, ci, comm.rank, comm.world, bounds=bounds).plan(comm)
            local_op = CsrOperator(_LocalCsr(rp, vals, shard), device)
        self.decomposition = "layers" if self.stencil else ("subdomain" if self.order is not None else "rows")
        super().__init__(local_op, partition, cfg, device=device)
        self.use_arena = False  # haloed blocks have their own (extended) sizes; _setup allocates them
        self.use_graphs = False  # iterations issue collectives: no graph capture
        self.cluster_ok = False  # the one-kernel cluster solve is a single-GPU path
        self.comm = comm
        self.shard = shard
        self.n_global = int(op.n)
        self.kmax = cfg.kmax if cfg.kmax is not None else 2 * self.n_global
        self.stag_window = max(20, self.kmax // 10) if self.retention == "restart" else 0
        self.n = self.shard.n_local  # every row-local kernel works on the local rows
        self.cache_aq = "auto"  # the lean scheme when the cached one does not fit the local HBM
        if self.stencil:
            self._desc = self._desc_rows(op, self.shard.row_begin, self.shard.row_end)
            interior, boundary = self.shard.row_ranges()
            self._desc_int = None if interior is None else self._desc_rows(op, *interior)
            self._desc_bnd = [self._desc_rows(op, a, b) for a, b in boundary]
        else:
            self.send_idx = {q: torch.from_numpy(v).to(self.device) for q, v in shard.send.items()}
        self._order_t = None if self.order is None else torch.from_numpy(self.order)

    @staticmethod
    def _desc_rows(op, r0, r1):
        desc = _lib.EkcgStencil()
        ctypes.memmove(ctypes.byref(desc), ctypes.byref(op._desc), ctypes.sizeof(desc))
        desc.row_begin, desc.row_end = r0, r1
        return desc

    def _global_to_local(self, v):
        """This rank's rows of a global vector (numpy or torch), in the engine's row order."""
        v = torch.as_tensor(v, dtype=torch.float64)
        if v.numel() != self.n_global:
            return v
        if self._order_t is not None:
            v = v[self._order_t.to(v.device)]
        return v[self.shard.row_begin:self.shard.row_end]

    # ------------------------------------------------------------ pointers
    def _lptr(self, ext, ld):
        """Local-row view of an extended (haloed) buffer."""
        return ext.data_ptr() + F64 * self.shard.lo * ld

    def _gptr_ext(self, ext, ld):
        """Global-row-addressed pointer into an extended buffer (stencil)."""
        return ext.data_ptr() + F64 * (self.shard.halo - self.shard.row_begin) * ld

    def _exchange(self, ext, ld):
        """Fill the halo rows of an extended block from the peers that own them."""
        self.comm.wait(self._exchange_start(ext, ld))

    def _exchange_start(self, ext, ld):
        if self.stencil:
            return self.comm.halo_exchange_start(ext, ld, self.shard)
        return self.comm.csr_exchange_start(ext, ld, self.shard, self.send_idx)

    def _exchange_apply(self, ext, col, ldx, y_loc, ldy, m, live):
        """Y_local = A X for columns [col, col + m) of the extended block `ext`:
        start the halo exchange, run the interior rows (no halo reads) while it is
        in flight, then wait and run the boundary rows.  The sends read the local
        rows and the receives write only the halo, so the interior product and the
        exchange touch disjoint data; the result equals one whole-shard product
        bit for bit (every row is computed by the same kernel arithmetic)."""
        works = self._exchange_start(ext, ldx)
        interior, boundary = self.shard.row_ranges()
        if not self.overlap or interior is None or works is None:
            self.comm.wait(works)
            self._apply_ext(ext, col, ldx, y_loc, ldy, m, live)
            return
        self._apply_rows(ext, col, ldx, y_loc, ldy, m, live, interior, self._desc_int if self.stencil else None)
        self.comm.wait(works)
        for j, rng in enumerate(boundary):
            self._apply_rows(ext, col, ldx, y_loc, ldy, m, live, rng, self._desc_bnd[j] if self.stencil else None)

    def _apply_rows(self, ext, col, ldx, y_loc, ldy, m, live, rng, desc):
        if self.stencil:
            _lib.call("ekcg_spmm_stencil", ctypes.byref(desc), self._gptr_ext(ext, ldx) + F64 * col, ldx,
                      y_loc - F64 * self.shard.row_begin * ldy, ldy, m, live, self.stream)
        else:
            self.op.apply_rows(rng[0], rng[1], ext.data_ptr() + F64 * col, ldx, y_loc, ldy, m, live, self.stream)

    def _apply_ext(self, ext, col, ldx, y_loc, ldy, m, live):
        """Y_local = A X for columns [col, col + m) of the extended block `ext`
        (halos filled) into the local-row pointer y_loc."""
        if self.stencil:
            self._stencil(self._gptr_ext(ext, ldx) + F64 * col, ldx, y_loc - F64 * self.shard.row_begin * ldy, ldy,
                          m, live)
        else:
            self.op.apply(ext.data_ptr() + F64 * col, ldx, y_loc, ldy, m, live, self.stream)

    def _gptr_loc(self, loc, ld):
        """Global-row-addressed pointer into a local (halo-free) buffer."""
        return loc.data_ptr() - F64 * self.shard.row_begin * ld

    def _stencil(self, x_gptr, ldx, y_gptr, ldy, m, live):
        _lib.call("ekcg_spmm_stencil", ctypes.byref(self._desc), x_gptr, ldx, y_gptr, ldy, m, live, self.stream)

    # --------------------------------------------------------------- setup
    def _setup(self):
        super()._setup()
        ext = self.shard.ext_rows
        mm = self.m_max
        f64 = dict(dtype=torch.float64, device=self.device)
        self.WA = torch.zeros(ext * mm, **f64)   # candidate / s-step chain (stencil input)
        if self.lean:  # WC carries A W, then W0 (stencil input); no WB
            self.WB = torch.empty(0, **f64)
            self.WC = torch.zeros(ext * mm, **f64)
        else:
            self.WB = torch.zeros(ext * mm, **f64)   # W0 (stencil input)
        self.fused_ok = True
        owner = self.partition.owner()[self.shard.row_begin:self.shard.row_end]
        self.owner_dev = torch.from_numpy(np.ascontiguousarray(owner, dtype=np.int32)).to(self.device)

    def _choose_lean(self, n, m):
        """The cached / lean decision must be the same on every rank (the
        schemes issue different collectives): lean if any rank needs it."""
        lean = super()._choose_lean(n, m)
        flag = torch.tensor([1.0 if lean else 0.0], dtype=torch.float64, device=self.device)
        self.comm.max_(flag)
        return bool(flag.item() > 0.0)

    def _new_block(self, width):
        ext = self.shard.ext_rows
        f64 = dict(dtype=torch.float64, device=self.device)
        if self.window is not None:
            slot = self.since_clear % self.window
            if slot not in self.slots:
                aq = None if self.lean else torch.empty(self.n * self.m_max, **f64)
                self.slots[slot] = (torch.zeros(ext * self.m_max, **f64), aq)
            q, aq = self.slots[slot]
        else:
            slot = -1
            q, aq = torch.zeros(ext * width, **f64), torch.empty(self.n * width, **f64)
        return _Block(q, aq, width, slot)

    def _allreduce(self, t):
        self.comm.allreduce_(t)

    # --------------------------------------------------------- residuals
    def _begin(self, b, x0):
        dev, st, sh = self.device, self.stream, self.shard
        self.b = self._global_to_local(b).to(dev).contiguous()
        self.x = torch.zeros(sh.ext_rows, dtype=torch.float64, device=dev)
        if x0 is not None:
            self.x[sh.lo:sh.lo + sh.n_local].copy_(self._global_to_local(x0).to(dev))
        self.r = torch.empty(self.n, dtype=torch.float64, device=dev)
        self._residual_sq(self.x, self.rho2, None, store_r=True)
        _lib.call("ekcg_start", self.ctrl.data_ptr(), self.rho2.data_ptr(), self.tol, self.history.data_ptr(), st)

    def _residual_sq(self, x, out, live, store_r=False):
        """out = |b - A x|^2 over all ranks (x extended with halos)."""
        st = self.stream
        self._exchange_apply(x, 0, 1, self.tmpv.data_ptr(), 1, 1, live)
        dst = self.r if store_r else self.tmpv
        _lib.call("ekcg_sub", self.b.data_ptr(), self.tmpv.data_ptr(), dst.data_ptr(), self.n, live, st)
        _lib.call("ekcg_sumsq", dst.data_ptr(), self.n, self.vpart.data_ptr(), live, st)
        _lib.call("ekcg_reduce", self.vpart.data_ptr(), self.vchunks, 1, out.data_ptr(), live, st)
        self.comm.allreduce_(out)

    def _final_metrics(self, x_star):
        self._residual_sq(self.x, self.tr2, None)
        true_res = float(torch.sqrt(self.tr2).item())
        rel = None
        if x_star is not None:
            sh = self.shard
            xs = self._global_to_local(x_star).to(self.device)
            xl = self.x[sh.lo:sh.lo + sh.n_local]
            sums = torch.stack([torch.sum((xl - xs) ** 2), torch.sum(xs ** 2)])
            self.comm.allreduce_(sums)
            rel = float(torch.sqrt(sums[0] / sums[1]).item())
        return true_res, rel

    def _output_x(self, numpy_io):
        sh = self.shard
        full = self.comm.gather_rows(self.x[sh.lo:sh.lo + sh.n_local].contiguous(), sh)
        if self._order_t is not None:  # back to the caller's row numbering
            out = torch.empty_like(full)
            out[self._order_t.to(full.device)] = full
            full = out
        if not numpy_io:
            return full
        out = torch.empty(full.numel(), dtype=torch.float64, pin_memory=True)  # see DeviceEngine._output_x
        out.copy_(full)
        return out.numpy()

    def _state(self, k, rho, tol1, numpy_io):
        raise NotImplementedError("on_iteration callbacks are not available on the sharded engine")

    # ----------------------------------------------------------- iteration
    def _enqueue_iteration_lean(self, k, tol1):
        """engine._enqueue_iteration_lean on a shard: w Q blocks + WA / WC, one
        operator application (with its halo exchange) per CGS2 pass."""
        cfg, n, st, live = self.cfg, self.n, self.stream, self.live
        if k > 1 and self.retention == "restart" and k % cfg.restart_j == 1:
            self._clear()
            self.restarts.append(k)
        elif (k > 1 and self.retention == "restart-tol" and tol1 < cfg.restart_tol
              and (not self.restarts or k > self.restarts[-1] + 1)):
            self._clear()
            self.restarts.append(k)
        m = t = self.t_cur
        d = len(self.retained)
        self._cur = (k, d, m)
        blk = self._new_block(m)
        lWA, lWC = self._lptr(self.WA, m), self._lptr(self.WC, m)
        lq = lambda b: self._lptr(b.q, b.width)
        base = self.arena.push([lq(b) for b in self.retained] + [lWA, lWC, lq(blk)])
        q_addr = lambda i: base + F64 * i
        WA_arr, WC_arr, NEW_arr = (base + F64 * (d + j) for j in range(3))
        fresh = not self.retained
        if fresh:
            _lib.call("ekcg_split", self.r.data_ptr(), self.owner_dev.data_ptr(), lWA, n, t, m, live, st)
        if d > 0:
            C = self._ensure("C", d * m * m)
            for _ in range(2):  # C = Q^T (A W), A symmetric (engine._enqueue_iteration_lean)
                self._exchange_apply(self.WA, 0, m, lWC, m, m, live)
                self._gram(q_addr(0), m, d, m, lWC, m, m, C.data_ptr(), tag="hist_gram")
                self.comm.allreduce_(C[: d * m * m])
                self._update(q_addr(0), m, d, m, C.data_ptr(), lWA, m, lWA, m, m, 1.0, -1.0, tag="hist_update")
        self._gram(WA_arr, m, 1, m, lWA, m, m, self.Graw.data_ptr(), tag="gram_self")
        self.comm.allreduce_(self.Graw[: m * m])
        _lib.call("ekcg_prechol", self.Graw.data_ptr(), m, self.S0.data_ptr(), live, k, 1e-14, st)
        self._tri_apply(WA_arr, m, self.S0.data_ptr(), lWC, m, m)  # W0 -> WC
        self._exchange_apply(self.WC, 0, m, lWA, m, m, live)  # A W0 -> WA (free)
        self._gram(WC_arr, m, 1, m, lWA, m, m, self.G.data_ptr(), tag="gram_aw")
        self.comm.allreduce_(self.G[: m * m])
        _lib.call("ekcg_cholinv", self.G.data_ptr(), m, self.S.data_ptr(), live, k, 1e-14, st)
        self._tri_apply(WC_arr, m, self.S.data_ptr(), lq(blk), m, m)
        self._gram(NEW_arr, m, 1, m, self.r.data_ptr(), 1, 1, self.alpha.data_ptr(), tag="gram_vec")
        self.comm.allreduce_(self.alpha[:m])
        self._exchange_apply(blk.q, 0, m, lWA, m, m, live)  # A W_k -> WA: the next candidate
        _lib.call("ekcg_xr_update", lq(blk), m, lWA, m, self.alpha.data_ptr(), m, self._lptr(self.x, 1),
                  self.r.data_ptr(), n, self.vpart.data_ptr(), live, st)
        _lib.call("ekcg_reduce", self.vpart.data_ptr(), self.vchunks, 1, self.rho2.data_ptr(), live, st)
        self.comm.allreduce_(self.rho2)
        self._append(blk)
        if k % self.every == 0:
            slot = k // self.every - 1
            self._ensure_checks(slot + 1)
            self._residual_sq(self.x, self.tr2, live)
            _lib.call("ekcg_store_norm", self.tr2.data_ptr(), self.checks.data_ptr(), slot, live, st)
        self._ensure_history(k + 1)
        _lib.call("ekcg_finish", self.ctrl.data_ptr(), self.rho2.data_ptr(), k, self.kmax, self.stag_window,
                  self.history.data_ptr(), st)
        self._account(k, d, m, fresh, t)

    def _enqueue_iteration(self, k, tol1):
        if self.lean:
            return self._enqueue_iteration_lean(k, tol1)
        cfg, n, st, live = self.cfg, self.n, self.stream, self.live
        if k > 1 and self.retention == "restart" and k % cfg.restart_j == 1:
            self._clear()
            self.restarts.append(k)
        elif (k > 1 and self.retention == "restart-tol" and tol1 < cfg.restart_tol
              and (not self.restarts or k > self.restarts[-1] + 1)):
            self._clear()
            self.restarts.append(k)
        t = self.t_cur
        m = self.s * t
        d = len(self.retained)
        self._cur = (k, d, m)
        newest = self.retained[-1] if self.retained else None
        blk = self._new_block(m)
        lWA, lWB = self._lptr(self.WA, m), self._lptr(self.WB, m)
        lq = lambda b: self._lptr(b.q, b.width)
        ptrs = [lq(b) for b in self.retained] + [b.aq.data_ptr() for b in self.retained] + [lWA, lWB, lq(blk)]
        base = self.arena.push(ptrs)
        q_addr = lambda i: base + F64 * i
        aq_addr = lambda i: base + F64 * (d + i)
        WA_arr, WB_arr, NEW_arr = (base + F64 * (2 * d + j) for j in range(3))

        # ---- candidate ----
        fresh = not self.retained
        W = lWA
        if fresh:
            _lib.call("ekcg_split", self.r.data_ptr(), self.owner_dev.data_ptr(), lWA, n, t, m, live, st)
            self._chain_sharded(m, t, live)
        elif self.s == 1:
            W = newest.aq.data_ptr()
        else:
            _lib.call("ekcg_copy_cols", newest.aq.data_ptr() + F64 * (newest.width - t), newest.width, lWA, m,
                      n, t, live, st)
            self._chain_sharded(m, t, live)

        # ---- CGS2 (aortho.py:89-95): local Grams, one allreduce per pass ----
        if d > 0:
            C = self._ensure("C", d * m * m)
            for _ in range(2):
                self._gram(aq_addr(0), m, d, m, W, m, m, C.data_ptr(), tag="hist_gram")
                self.comm.allreduce_(C[: d * m * m])
                self._update(q_addr(0), m, d, m, C.data_ptr(), W, m, lWA, m, m, 1.0, -1.0, tag="hist_update")
                W = lWA

        # ---- Pre-CholQR ----
        self._gram(WA_arr, m, 1, m, lWA, m, m, self.Graw.data_ptr(), tag="gram_self")
        self.comm.allreduce_(self.Graw[: m * m])
        _lib.call("ekcg_prechol", self.Graw.data_ptr(), m, self.S0.data_ptr(), live, k, 1e-14, st)
        self._tri_apply(WA_arr, m, self.S0.data_ptr(), lWB, m, m)
        fused = m in (8, 16, 32, 64)
        # same kernel choice as DeviceEngine: the fused stencil kernels only for
        # m <= 16, the plane-marching stencil + DMMA kernels above (CSR: unfused)
        fused_st = fused and m <= 16 and self.stencil
        part = self._ensure("part", max(self.fused_part, 1)) if fused else None
        if fused_st:
            self._exchange(self.WB, m)
            _lib.call("ekcg_stencil_cholinv", ctypes.byref(self._desc), self._gptr_ext(self.WB, m), m, m,
                      part.data_ptr(), self.counter.data_ptr(), self.G.data_ptr(), live, k, 1e-14, 0, st)
        else:
            self._exchange_apply(self.WB, 0, m, self.WC.data_ptr(), m, m, live)
            self._gram(WB_arr, m, 1, m, self.WC.data_ptr(), m, m, self.G.data_ptr(), tag="gram_aw")
        self.comm.allreduce_(self.G[: m * m])
        _lib.call("ekcg_cholinv", self.G.data_ptr(), m, self.S.data_ptr(), live, k, 1e-14, st)
        if fused_st:
            _lib.call("ekcg_update_vec", WB_arr, m, self.S.data_ptr(), lq(blk), m, m, n, self.r.data_ptr(),
                      part.data_ptr(), self.counter.data_ptr(), self.alpha.data_ptr(), live, st)
        else:
            self._tri_apply(WB_arr, m, self.S.data_ptr(), lq(blk), m, m)
            self._gram(NEW_arr, m, 1, m, self.r.data_ptr(), 1, 1, self.alpha.data_ptr(), tag="gram_vec")
        self.comm.allreduce_(self.alpha[:m])

        # ---- AW_k = A W_k and the iterate update ----
        if fused_st:
            self._exchange(blk.q, m)
            _lib.call("ekcg_stencil_xr", ctypes.byref(self._desc), self._gptr_ext(blk.q, m), m,
                      self._gptr_loc(blk.aq, m), m, m, self.alpha.data_ptr(), self._gptr_ext(self.x, 1),
                      self._gptr_loc(self.r, 1), part.data_ptr(), self.counter.data_ptr(), live, k, self.kmax,
                      self.stag_window, self.history.data_ptr(), 0, self.rho2.data_ptr(), st)
        else:
            self._exchange_apply(blk.q, 0, m, blk.aq.data_ptr(), m, m, live)
            _lib.call("ekcg_xr_update", lq(blk), m, blk.aq.data_ptr(), m, self.alpha.data_ptr(), m,
                      self._lptr(self.x, 1), self.r.data_ptr(), n, self.vpart.data_ptr(), live, st)
            _lib.call("ekcg_reduce", self.vpart.data_ptr(), self.vchunks, 1, self.rho2.data_ptr(), live, st)
        self.comm.allreduce_(self.rho2)
        self._append(blk)
        if k % self.every == 0:
            slot = k // self.every - 1
            self._ensure_checks(slot + 1)
            self._residual_sq(self.x, self.tr2, live)
            _lib.call("ekcg_store_norm", self.tr2.data_ptr(), self.checks.data_ptr(), slot, live, st)
        self._ensure_history(k + 1)
        _lib.call("ekcg_finish", self.ctrl.data_ptr(), self.rho2.data_ptr(), k, self.kmax, self.stag_window,
                  self.history.data_ptr(), st)
        self._account(k, d, m, fresh, t)

    def _chain_sharded(self, m, t, live):
        for i in range(1, self.s):
            self._exchange_apply(self.WA, (i - 1) * t, m, self._lptr(self.WA, m) + F64 * i * t, m, t, live)
