"""Device engine: the `_run_engine` loop (solvers.py:319-428) as a stream of
sm_100a kernel launches.

One iteration (SRE-CG2, d retained blocks, width m = s*t) issues:

  candidate   W = A W_{k-1} (cached, no copy) | split(r) | s-step chain | MSDO
  CGS2 x 2    C = [AQ_1..AQ_d]^T W (DMMA split-K Gram) ; W <- W - sum Q_i C_i
  Pre-CholQR  Graw = W^T W ; S0 = D^-1 chol(sym(D^-1 Graw D^-1))^-1 ; W0 = W S0
  A-CholQR    G = W0^T (A W0) ; S = chol(sym G)^-1 ; W_k = W0 S ; AW_k = A W_k
  update      alpha = W_k^T r ; x += W_k alpha ; r -= AW_k alpha ; rho = |r|
  finish      history[k] = rho, stop test, stagnation guard (device)

Every launch is gated on a device `live` flag that the Cholesky kernels
(breakdown) and the finish kernel (converged / maxiter / stagnated) clear,
so the host enqueues iterations ahead and polls the control block once per
batch instead of synchronising every iteration.  The retained history is a
ring of `trunc` slots in HBM (truncated / SRE-CG), or one block pair per
iteration (full retention); the new block overwrites the oldest slot only
after the second Gram-Schmidt pass has consumed it.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np
import torch

from . import _lib
from .device import get_device
from .operators import as_operator
from .solvers import BasisStore, ConvergenceReport

_STATUS = {1: "converged", 2: "maxiter", 3: "breakdown", 4: "stagnated"}
F64 = 8


class _PtrArena:
    """Write-once device arena of block-pointer arrays (the kernels take
    `const double* const*`).  Each iteration pushes its pointer lists with one
    async H2D copy from pinned memory; a region is rewritten only after a
    stream sync."""

    def __init__(self, device, capacity=1 << 15):
        self.device = device
        self.cap = capacity
        self._alloc(capacity)

    def _alloc(self, cap):
        self.floor = 0  # regions below `floor` belong to captured CUDA graphs
        self.cap = cap
        self.host = torch.empty(cap, dtype=torch.int64, pin_memory=True)
        self.hnp = self.host.numpy()
        self.dev = torch.empty(cap, dtype=torch.int64, device=self.device)
        self.cur = 0

    def push(self, ptrs):
        L = len(ptrs)
        if self.cur + L > self.cap:
            torch.cuda.current_stream(self.device).synchronize()
            if self.floor + L > self.cap:
                raise RuntimeError("pointer arena exhausted by captured graphs")
            self.cur = self.floor
        s = self.cur
        self.hnp[s:s + L] = ptrs
        self.dev[s:s + L].copy_(self.host[s:s + L], non_blocking=True)
        self.cur += L
        return self.dev.data_ptr() + F64 * s


class _Block:
    __slots__ = ("q", "aq", "width", "slot")

    def __init__(self, q, aq, width, slot):
        self.q, self.aq, self.width, self.slot = q, aq, width, slot


class DeviceEngine:
    """One solve of an enlarged-CG method on one GPU."""

    def __init__(self, A, partition, cfg, device=None):
        self.device = get_device(device)
        self.op = as_operator(A, self.device)
        self.n = int(self.op.n)
        self.partition = partition
        self.cfg = cfg
        self.method = cfg.method
        self.s = int(cfg.s)
        self.retention = "trunc" if cfg.method == "sre-cg" else cfg.retention
        self.window = cfg.effective_window()
        self.kmax = cfg.kmax if cfg.kmax is not None else 2 * self.n
        self.every = int(cfg.true_residual_every)
        self.tol = float(cfg.tol)
        self.stag_window = max(20, self.kmax // 10) if self.retention == "restart" else 0
        self.sync_mode = False
        self.max_lookahead = 16
        # size run-ahead batches from the residual decay seen in the snapshots, so that
        # few gated (no-op) iterations are queued past convergence
        self.predict_batches = True
        self.kernel_timer = None  # optional hook: (name, callable) -> runs callable
        self.no_fuse = False      # force the unfused kernel sequence (tests / A-B timing)
        # fused stages in use when the operator/width allow: "prechol" (update2 + Graw + S0),
        # "cholinv" (A W0 + G + S), "vec" (W0 S + alpha), "xr" (A W_k + x/r + finish)
        self.fuse = {"cholinv", "vec", "xr"}
        # small (launch-latency-bound) blocks also fuse the second CGS2 update with Graw and the
        # Pre-CholQR factor: config 1 10.2k -> 11.9k it/s; on config 2 (4.2 M block entries) the
        # fused kernel is slower (tools/ab_graphs.py --prechol)
        self.fuse_prechol_max = 1 << 20
        # cache A Q next to every retained Q (reference scheme, aortho.py:82-87) or
        # recompute the projections as Q^T (A W) with A symmetric ("lean": w + 2
        # blocks of HBM instead of 2w + 3; two extra operator applications per
        # iteration).  "auto" picks lean only when the cached scheme does not fit.
        self.cache_aq = "auto"
        # split block-Jacobi preconditioner, "modified" mode (solvers.py:326-339)
        self.pc = None
        self.pc_aligned = True
        self.norm_pc = None  # explicit-hat mode: residual norms are |L r_hat| (solvers.py:305-306)
        self.notes_init = []
        F = cfg.preconditioner
        if F is not None and cfg.precond_mode == "modified":
            from .precond import DevicePreconditioner, aligned_with
            self.pc = F if isinstance(F, DevicePreconditioner) else DevicePreconditioner(F, self.device)
            self.pc_aligned = aligned_with(self.pc.host, partition)
            if not self.pc_aligned:
                self.notes_init.append("preconditioner blocks not aligned with partition subdomains; "
                                       "using explicit split application")
        # replay steady-state iterations of truncated windows from CUDA graphs (one per ring
        # phase; iteration numbers are read on the device).  "auto": for small blocks
        # (n m <= 2^20), where the Python enqueue of an iteration (~80 us) is as long as the
        # GPU's (~84 us at config 1) and the queue would drain at batch boundaries; a replay
        # costs ~10 us of host time.  Large blocks gain nothing from it.
        self.use_graphs = "auto"
        self._capturing = False
        self._slab, self._slab_off = None, 0
        # NVTX ranges per iteration and per tagged launch (host cost only when on)
        self.nvtx = os.environ.get("EKCG_NVTX", "0") == "1"
        self.use_arena = True  # one allocation for all of a truncated window's blocks (see _setup)
        # whole solve in one thread-block-cluster kernel (csrc/cluster_solve.cu) for small
        # truncated-window problems: "auto" (n t up to ~2e5, where an iteration of separate
        # launches is latency-bound), True (whenever the kernel applies) or False
        self.use_cluster = "auto"
        self.cluster_ok = True  # False in the sharded engine
        self.ran_cluster = False
        self.cluster_ticks = None  # optional int64[20] device tensor: per-phase SM cycles of CTA 0

    # ------------------------------------------------------------------ setup
    def _setup(self):
        dev, n = self.device, self.n
        self.stream = torch.cuda.current_stream(dev).cuda_stream
        self.t_cur = int(self.partition.t)
        self.m_max = self.s * self.t_cur
        mm = self.m_max
        f64 = dict(dtype=torch.float64, device=dev)
        self.lean = self._choose_lean(n, mm)
        # Truncated windows: every n x m block of the solve (WA, WB, WC and the ring slots) is a slice of
        # ONE allocation, so the caching allocator hands the same segment back to the next solve of the
        # same size -- separately allocated 34 GB blocks fragment it (config 5: the second solve in a
        # process could not find a 32 GiB hole in 31.5 GiB of free cache).
        self._arena, self._arena_next = None, 0
        if self.window is not None and self.use_arena:
            nblk = (2 if self.lean else 3) + self.window * (1 if self.lean else 2)
            self._arena = torch.empty(nblk * self._span(n * mm), **f64)
            take = self._arena_block
        else:
            take = lambda numel: torch.empty(numel, **f64)  # noqa: E731
        self.WA = take(n * mm)
        self.WB = torch.empty(0, **f64) if self.lean else take(n * mm)
        self.WC = take(n * mm)
        self.tmpv = torch.empty(n, **f64)
        self.tmpv2 = torch.empty(n, **f64)
        self.tmpv3 = torch.empty(n, **f64)
        self.Graw = torch.empty(mm * mm, **f64)
        self.G = torch.empty(mm * mm, **f64)
        self.S0 = torch.empty(mm * mm, **f64)
        self.S = torch.empty(mm * mm, **f64)
        self.alpha = torch.empty(mm, **f64)
        self.beta = torch.empty(mm, **f64)
        self.rho2 = torch.empty(1, **f64)
        self.tr2 = torch.empty(1, **f64)
        self.vchunks = _lib.query("ekcg_vec_chunks", n)
        self.vpart = torch.empty(self.vchunks, **f64)
        self.part = torch.empty(1 << 16, **f64)
        self.C = torch.empty(1 << 12, **f64)
        self.ctrl = torch.zeros(_lib.query("ekcg_ctrl_bytes"), dtype=torch.uint8, device=dev)
        self.ctrl_host = torch.empty(self.ctrl.numel(), dtype=torch.uint8, pin_memory=True)
        self.snap_bufs = [torch.empty(self.ctrl.numel(), dtype=torch.uint8, pin_memory=True) for _ in range(3)]
        self.live = self.ctrl.data_ptr()
        hist_len = min(self.kmax, 1 << 20) + 1 if self.window is not None else min(self.kmax, 4096) + 1
        self.history = torch.zeros(hist_len, **f64)
        self.checks = torch.zeros(max(1, (hist_len - 1) // self.every + 1), **f64)
        self.arena = _PtrArena(dev)
        self.owner_dev = self.partition.device_owner(dev)
        self.part_obj = self.partition
        self.retained = []
        self.slots = {}
        self.since_clear = 0
        self.cols = 0
        self.peak = 0
        self.restarts = []
        self.switch_iteration = None
        self.gram_chunks = {}
        self.launch_k = []
        self.counter = torch.zeros(64, dtype=torch.int32, device=dev)  # EKCG_FUSED_COUNTERS
        from .operators import StencilOperator
        self.fused_ok = isinstance(self.op, StencilOperator) and not self.no_fuse
        self.fused_part = _lib.query("ekcg_fused_partials", n, mm)

    def _choose_lean(self, n, m):
        eligible = (self.window is not None and self.s == 1 and self.method in ("sre-cg2", "sre-cg")
                    and self.cfg.switch_tol is None and self.pc is None)
        if self.cache_aq is True or not eligible:
            if self.cache_aq is False and not eligible:
                raise ValueError("the lean (no A Q cache) scheme needs a truncation window, s = 1, "
                                 "an SRE method and no flexible switch")
            return False
        if self.cache_aq is False:
            return True
        block = 8.0 * n * m
        cached = (2 * self.window + 3) * block + 6 * 8.0 * n
        if cached < (1 << 30):  # small solves: no cudaMemGetInfo round trip (~0.2 ms of a 6 ms config-1 call)
            return False
        free, _ = torch.cuda.mem_get_info(self.device)
        return cached > 0.92 * free

    @staticmethod
    def _span(numel):
        return (numel + 31) // 32 * 32  # slices start on 256-B boundaries (TMA / 256-bit loads)

    def _arena_block(self, numel):
        """The next n x m_max slice of the solve's block arena."""
        v = self._arena[self._arena_next:self._arena_next + numel]
        self._arena_next += self._span(numel)
        return v

    def _ensure(self, name, numel):
        buf = getattr(self, name)
        if buf.numel() < numel:
            buf = torch.empty(max(numel, 2 * buf.numel()), dtype=buf.dtype, device=self.device)
            setattr(self, name, buf)
        return buf

    def _karg(self, k):
        """Iteration number as a kernel argument: <= 0 inside a graph capture
        (the kernels then read ctrl->k_done + 1 on the device)."""
        return -1 if self._capturing else k

    def _graph_eligible(self):
        want = (self.n * self.m_max <= (1 << 20)) if self.use_graphs == "auto" else bool(self.use_graphs)
        return (want and self.kernel_timer is None and self.window is not None
                and self.retention == "trunc" and self.cfg.switch_tol is None
                and self.method in ("sre-cg2", "sre-cg") and self.kmax + 1 <= self.history.numel())

    def _host_step(self, k):
        """Host bookkeeping of a replayed iteration (what _enqueue_iteration does besides launching)."""
        m = self.s * self.t_cur
        d = len(self.retained)
        self._cur = (k, d, m)
        blk = self._new_block(m)
        self._append(blk)
        self._account(k, d, m, False, self.t_cur)

    def _capture_iteration(self, k):
        """Capture iteration k (a steady-state ring phase) into a CUDA graph; returns it (not yet replayed)."""
        g = torch.cuda.CUDAGraph()
        m, d = self.s * self.t_cur, len(self.retained)
        self._ensure("part", max(self.fused_part, self._chunks(d, m, m) * d * m * m, self._chunks(1, m, m) * m * m,
                                 self._chunks(1, m, 1) * m, self._chunks(1, m, m) * m * m))
        self._ensure("C", d * m * m + 1)
        if self.arena.cur + 4 * (2 * d + 8) > self.arena.cap:  # never wrap while capturing
            torch.cuda.current_stream(self.device).synchronize()
            self.arena.cur = self.arena.floor
        saved = self.stream
        self._capturing = True
        try:
            with torch.cuda.graph(g):
                self.stream = torch.cuda.current_stream(self.device).cuda_stream
                self._enqueue_iteration(k, 1.0)
        finally:
            self._capturing = False
            self.stream = saved
        self.arena.floor = self.arena.cur
        return g

    def _chunks(self, d, m1, m2):
        key = (d, m1, m2)
        c = self.gram_chunks.get(key)
        if c is None:
            c = _lib.query("ekcg_gram_chunks", self.n, d, m1, m2)
            self.gram_chunks[key] = c
        return c

    # ---------------------------------------------------------- primitives
    def _gram(self, xs_addr, ldx, d, m1, y_ptr, ldy, m2, out_ptr, tag="gram"):
        """out (d*m1*m2) = [X_i^T Y] via split-K partials + fixed-order reduce."""
        chunks = self._chunks(d, m1, m2)
        part = self._ensure("part", chunks * d * m1 * m2)
        run = lambda: _lib.call("ekcg_gram", xs_addr, ldx, d, m1, y_ptr, ldy, m2, self.n, part.data_ptr(),
                                self.live, self.stream)
        self._timed(tag, run)
        _lib.call("ekcg_reduce", part.data_ptr(), chunks, d * m1 * m2, out_ptr, self.live, self.stream)

    def _update(self, qs_addr, ldq, d, m1, c_ptr, win_ptr, ldwi, wout_ptr, ldwo, m2, beta, sign, tag="update"):
        run = lambda: _lib.call("ekcg_block_update", qs_addr, ldq, d, m1, c_ptr, win_ptr, ldwi, wout_ptr, ldwo,
                                m2, beta, sign, self.n, self.live, self.stream)
        self._timed(tag, run)

    def _tri_apply(self, w_arr, ldw, s_ptr, out_ptr, ldo, m, tag="tri_apply"):
        """out = W S with S upper triangular (W R^-1 of aortho.py:106,109)."""
        self._timed(tag, lambda: _lib.call("ekcg_tri_apply", w_arr, ldw, s_ptr, out_ptr, ldo, m, self.n, self.live,
                                           self.stream))

    def _apply_op(self, x_ptr, ldx, y_ptr, ldy, m, tag="spmm", live=-1):
        gate = self.live if live == -1 else live
        self._timed(tag, lambda: self.op.apply(x_ptr, ldx, y_ptr, ldy, m, gate, self.stream))

    def _timed(self, tag, fn):
        if self.nvtx:
            torch.cuda.nvtx.range_push(tag)
        if self.kernel_timer is None:
            fn()
        else:
            self.kernel_timer(tag, fn)
        if self.nvtx:
            torch.cuda.nvtx.range_pop()

    def _enqueue(self, k, tol1):
        """One iteration's launches, inside an NVTX range when EKCG_NVTX=1 (nsys timelines)."""
        if not self.nvtx:
            return self._enqueue_iteration(k, tol1)
        torch.cuda.nvtx.range_push(f"iteration {k}")
        try:
            return self._enqueue_iteration(k, tol1)
        finally:
            torch.cuda.nvtx.range_pop()

    # -------------------------------------------------------------- store
    def _new_block(self, width):
        """Storage for W_k / AW_k.  Ring slot (trunc windows) or fresh pair (full)."""
        n = self.n
        if self.window is not None:
            slot = self.since_clear % self.window
            if slot not in self.slots:
                f64 = dict(dtype=torch.float64, device=self.device)
                take = self._arena_block if self._arena is not None else (
                    lambda numel: torch.empty(numel, **f64))  # noqa: E731
                q = take(n * self.m_max)
                aq = None if self.lean else take(n * self.m_max)
                self.slots[slot] = (q, aq)
            qbuf, aqbuf = self.slots[slot]
        else:
            slot = -1
            qbuf, aqbuf = self._carve(n * width), self._carve(n * width)
        return _Block(qbuf, aqbuf, width, slot)

    def _carve(self, numel):
        """A fresh n x width block for full retention, carved from slabs of about
        1 GiB: one allocation per slab instead of two per iteration, so a cold
        caching allocator costs a few cudaMalloc calls per solve, not hundreds.
        Views start on 256-B boundaries; blocks of >= 128 MiB are allocated alone."""
        f64 = dict(dtype=torch.float64, device=self.device)
        if numel * 8 >= (1 << 27):
            return torch.empty(numel, **f64)
        span = (numel + 31) // 32 * 32
        if self._slab is None or self._slab_off + span > self._slab.numel():
            per = max(1, (1 << 30) // (span * 8))
            self._slab = torch.empty(per * span, **f64)
            self._slab_off = 0
        v = self._slab[self._slab_off:self._slab_off + numel]
        self._slab_off += span
        return v

    def _append(self, blk):
        self.retained.append(blk)
        self.since_clear += 1
        self.cols += blk.width
        self.peak = max(self.peak, self.cols)
        if self.window is not None:
            while len(self.retained) > self.window:
                old = self.retained.pop(0)
                self.cols -= old.width

    def _clear(self):
        self.retained = []
        self.since_clear = 0
        self.cols = 0

    # ------------------------------------------------------------ iteration
    def _width_groups(self):
        groups, start = [], 0
        for i in range(1, len(self.retained) + 1):
            if i == len(self.retained) or self.retained[i].width != self.retained[start].width:
                groups.append((start, i, self.retained[start].width))
                start = i
        return groups

    def _enqueue_iteration(self, k, tol1):
        if self.lean:
            return self._enqueue_iteration_lean(k, tol1)
        cfg, n = self.cfg, self.n
        st, live = self.stream, self.live
        # restart policies (solvers.py:358-364)
        if k > 1 and self.retention == "restart" and k % cfg.restart_j == 1:
            self._clear()
            self.restarts.append(k)
        elif (k > 1 and self.retention == "restart-tol" and tol1 < cfg.restart_tol
              and (not self.restarts or k > self.restarts[-1] + 1)):
            self._clear()
            self.restarts.append(k)
        switched = False
        if (cfg.switch_tol is not None and self.switch_iteration is None and k > 1
                and tol1 < cfg.switch_tol):
            self.part_obj = self.part_obj.halve()
            self.owner_dev = self.part_obj.device_owner(self.device)
            self.t_cur //= 2
            self.switch_iteration = k
            switched = True

        t = self.t_cur
        m = self.s * t
        d = len(self.retained)
        self._cur = (k, d, m)  # read by optional kernel timers
        groups = self._width_groups()
        newest = self.retained[-1] if self.retained else None
        blk = self._new_block(m)
        WA, WB, WC = self.WA.data_ptr(), self.WB.data_ptr(), self.WC.data_ptr()
        ptrs = [b.q.data_ptr() for b in self.retained] + [b.aq.data_ptr() for b in self.retained]
        ptrs += [WA, WB, blk.q.data_ptr(), newest.aq.data_ptr() if newest is not None else 0]
        base = self.arena.push(ptrs)
        q_addr = lambda i: base + F64 * i
        aq_addr = lambda i: base + F64 * (d + i)
        WA_arr, WB_arr, NEW_arr, NEWEST_AQ_arr = (base + F64 * (2 * d + j) for j in range(4))

        # ---- candidate block (solvers.py:366-382) ----
        fresh = switched or not self.retained
        W = WA
        pc = self.pc
        if fresh or self.method == "modified-msdo-cg":
            self._candidate_split(WA, t, m)
            self._chain(WA, m, t)
        elif self.method in ("sre-cg2", "sre-cg"):
            if pc is not None:  # chain_next = M^-1 A W_{k-1} (solvers.py:338-339)
                self._minv(newest.aq.data_ptr(), newest.width, WA, m, m)
            elif self.s == 1:
                W = newest.aq.data_ptr()  # W_k = A W_{k-1}: read the cached product in place
            else:
                src = newest.aq.data_ptr() + F64 * (newest.width - t)
                _lib.call("ekcg_copy_cols", src, newest.width, WA, m, n, t, live, st)
                self._chain(WA, m, t)
        elif pc is None:  # msdo-cg: split(r) + W_prev diag(-(AW_prev^T r))
            self._gram(NEWEST_AQ_arr, newest.width, 1, newest.width, self.r.data_ptr(), 1, 1,
                       self.beta.data_ptr(), tag="gram_vec")
            _lib.call("ekcg_split_axpy", self.r.data_ptr(), self.owner_dev.data_ptr(), newest.q.data_ptr(),
                      newest.width, self.beta.data_ptr(), -1.0, WA, n, t, m, live, st)
        else:  # preconditioned msdo-cg: M^-1 split(r) + W_prev diag(-(AW_prev^T M^-1 r))
            self._minv(self.r.data_ptr(), 1, self.tmpv2.data_ptr(), 1, 1)
            self._gram(NEWEST_AQ_arr, newest.width, 1, newest.width, self.tmpv2.data_ptr(), 1, 1,
                       self.beta.data_ptr(), tag="gram_vec")
            self._candidate_split(WA, t, m)
            _lib.call("ekcg_axpy_cols", WA, m, newest.q.data_ptr(), newest.width, self.beta.data_ptr(), -1.0, n, t,
                      live, st)

        fused = (self.fused_ok and m in (8, 16, 32, 64)
                 and all(b.width == m for b in self.retained))
        if fused:
            part = self._ensure("part", self.fused_part)
        # ---- CGS2 against the retained history (aortho.py:89-95) ----
        have_s0 = False
        if d > 0:
            csz = sum((e - s0) * wg * m for s0, e, wg in groups)
            C = self._ensure("C", csz)
            for pas in range(2):
                off = 0
                for s0, e, wg in groups:  # all coefficients from the same W (classical GS)
                    self._gram(aq_addr(s0), wg, e - s0, wg, W, m, m, C.data_ptr() + F64 * off, tag="hist_gram")
                    off += (e - s0) * wg * m
                if fused and pas == 1 and ("prechol" in self.fuse or n * m <= self.fuse_prechol_max):
                    # W'' = W' - Q C2 fused with Graw = W''^T W'' and the Pre-CholQR factor
                    self._timed("hist_update", lambda: _lib.call(
                        "ekcg_update_prechol", q_addr(0), m, d, C.data_ptr(), WA, m, WA, m, m, n,
                        part.data_ptr(), self.counter.data_ptr(), self.S0.data_ptr(), live, self._karg(k), 1e-14, st))
                    have_s0 = True
                    break
                off = 0
                win = W
                for s0, e, wg in groups:
                    self._update(q_addr(s0), wg, e - s0, wg, C.data_ptr() + F64 * off, win, m, WA, m, m,
                                 1.0, -1.0, tag="hist_update")
                    win = WA
                    off += (e - s0) * wg * m
                W = WA

        # ---- Pre-CholQR (aortho.py:98-110) ----
        if not have_s0:
            self._gram(WA_arr, m, 1, m, WA, m, m, self.Graw.data_ptr(), tag="gram_self")
            _lib.call("ekcg_prechol", self.Graw.data_ptr(), m, self.S0.data_ptr(), live, self._karg(k), 1e-14, st)
        self._tri_apply(WA_arr, m, self.S0.data_ptr(), WB, m, m)
        finish_now = (k % self.every != 0)
        if fused and "cholinv" in self.fuse and m <= 16:
            # G = W0^T A W0 (A W0 never written) + A-CholQR factor S.  For m >= 32
            # the unfused stencil + DMMA Gram is faster (kernel_times.py --fused).
            self._timed("spmm_gram", lambda: _lib.call(
                "ekcg_stencil_cholinv", self.op.desc_ref(), WB, m, m, part.data_ptr(), self.counter.data_ptr(),
                self.S.data_ptr(), live, self._karg(k), 1e-14, 1, st))
        else:
            self._apply_op(WB, m, WC, m, m)
            self._gram(WB_arr, m, 1, m, WC, m, m, self.G.data_ptr(), tag="gram_aw")
            _lib.call("ekcg_cholinv", self.G.data_ptr(), m, self.S.data_ptr(), live, self._karg(k), 1e-14, st)
        if fused and "vec" in self.fuse and m <= 16:
            # W_k = W0 S + alpha = W_k^T r (for m >= 32 the smem-staged update + X^T r kernel is faster)
            self._timed("tri_alpha", lambda: _lib.call(
                "ekcg_update_vec", WB_arr, m, self.S.data_ptr(), blk.q.data_ptr(), m, m, n, self.r.data_ptr(),
                part.data_ptr(), self.counter.data_ptr(), self.alpha.data_ptr(), live, st))
        else:
            self._tri_apply(WB_arr, m, self.S.data_ptr(), blk.q.data_ptr(), m, m)
            self._gram(NEW_arr, m, 1, m, self.r.data_ptr(), 1, 1, self.alpha.data_ptr(), tag="gram_vec")
        # m >= 32: the plane-marching stencil + xr_update beats the fused row kernel
        xr_fused = fused and "xr" in self.fuse and m <= 16
        if xr_fused:
            # AW_k = A W_k + x/r update + |r|^2 + end-of-iteration bookkeeping (solvers.py:394-415)
            self._ensure_history(k + 1)
            self._timed("spmm_xr", lambda: _lib.call(
                "ekcg_stencil_xr", self.op.desc_ref(), blk.q.data_ptr(), m, blk.aq.data_ptr(), m, m,
                self.alpha.data_ptr(), self.x.data_ptr(), self.r.data_ptr(), part.data_ptr(),
                self.counter.data_ptr(), live, self._karg(k), self.kmax, self.stag_window, self.history.data_ptr(),
                1 if finish_now else 0, self.rho2.data_ptr(), st))
        else:
            self._apply_op(blk.q.data_ptr(), m, blk.aq.data_ptr(), m, m)
            # ---- iterate update (solvers.py:394-399) ----
            self._timed("xr_update", lambda: _lib.call(
                "ekcg_xr_update", blk.q.data_ptr(), m, blk.aq.data_ptr(), m, self.alpha.data_ptr(), m,
                self.x.data_ptr(), self.r.data_ptr(), n, self.vpart.data_ptr(), live, st))
            _lib.call("ekcg_reduce", self.vpart.data_ptr(), self.vchunks, 1, self.rho2.data_ptr(), live, st)
            if self.norm_pc is not None:  # |L r_hat| instead of |r_hat|
                _lib.call("ekcg_sumsq", self._normed(self.r, live), n, self.vpart.data_ptr(), live, st)
                _lib.call("ekcg_reduce", self.vpart.data_ptr(), self.vchunks, 1, self.rho2.data_ptr(), live, st)
        self._append(blk)
        if not finish_now:  # true-residual drift log (solvers.py:401-402)
            slot = k // self.every - 1
            self._ensure_checks(slot + 1)
            self._residual_sq(self.x, self.tr2, live)
            _lib.call("ekcg_store_norm", self.tr2.data_ptr(), self.checks.data_ptr(), slot, live, st)
        if not (xr_fused and finish_now):
            self._ensure_history(k + 1)
            _lib.call("ekcg_finish", self.ctrl.data_ptr(), self.rho2.data_ptr(), self._karg(k), self.kmax, self.stag_window,
                      self.history.data_ptr(), st)
        self._account(k, d, m, fresh, t)

    def _enqueue_iteration_lean(self, k, tol1):
        """One iteration without cached A Q (HBM: w Q blocks + 2 scratch).

        WA carries the candidate A W_{k-1} between iterations; the CGS2
        coefficients are C = Q_i^T (A W) (A symmetric), so each pass applies the
        operator once (into WC) instead of reading cached A Q_i.
        """
        cfg, n = self.cfg, self.n
        st, live = self.stream, self.live
        if k > 1 and self.retention == "restart" and k % cfg.restart_j == 1:
            self._clear()
            self.restarts.append(k)
        elif (k > 1 and self.retention == "restart-tol" and tol1 < cfg.restart_tol
              and (not self.restarts or k > self.restarts[-1] + 1)):
            self._clear()
            self.restarts.append(k)
        t = self.t_cur
        m = t
        d = len(self.retained)
        self._cur = (k, d, m)
        blk = self._new_block(m)
        WA, WC = self.WA.data_ptr(), self.WC.data_ptr()
        ptrs = [b.q.data_ptr() for b in self.retained] + [WA, WC, blk.q.data_ptr()]
        base = self.arena.push(ptrs)
        q_addr = lambda i: base + F64 * i
        WA_arr, WC_arr, NEW_arr = (base + F64 * (d + j) for j in range(3))
        fresh = not self.retained
        if fresh:
            _lib.call("ekcg_split", self.r.data_ptr(), self.owner_dev.data_ptr(), WA, n, t, m, live, st)
        fused = self.fused_ok and m in (8, 16, 32, 64)
        part = self._ensure("part", self.fused_part) if fused else None
        if d > 0:
            C = self._ensure("C", d * m * m)
            for _ in range(2):
                self._apply_op(WA, m, WC, m, m, tag="spmm_proj")
                self._gram(q_addr(0), m, d, m, WC, m, m, C.data_ptr(), tag="hist_gram")
                self._update(q_addr(0), m, d, m, C.data_ptr(), WA, m, WA, m, m, 1.0, -1.0, tag="hist_update")
        self._gram(WA_arr, m, 1, m, WA, m, m, self.Graw.data_ptr(), tag="gram_self")
        _lib.call("ekcg_prechol", self.Graw.data_ptr(), m, self.S0.data_ptr(), live, self._karg(k), 1e-14, st)
        self._tri_apply(WA_arr, m, self.S0.data_ptr(), WC, m, m)  # W0 -> WC
        if fused and m <= 16:
            self._timed("spmm_gram", lambda: _lib.call(
                "ekcg_stencil_cholinv", self.op.desc_ref(), WC, m, m, part.data_ptr(), self.counter.data_ptr(),
                self.S.data_ptr(), live, self._karg(k), 1e-14, 1, st))
        else:
            self._apply_op(WC, m, WA, m, m)  # A W0 -> WA (free)
            self._gram(WC_arr, m, 1, m, WA, m, m, self.G.data_ptr(), tag="gram_aw")
            _lib.call("ekcg_cholinv", self.G.data_ptr(), m, self.S.data_ptr(), live, self._karg(k), 1e-14, st)
        if fused and m <= 16:
            self._timed("tri_alpha", lambda: _lib.call(
                "ekcg_update_vec", WC_arr, m, self.S.data_ptr(), blk.q.data_ptr(), m, m, n, self.r.data_ptr(),
                part.data_ptr(), self.counter.data_ptr(), self.alpha.data_ptr(), live, st))
        else:
            self._tri_apply(WC_arr, m, self.S.data_ptr(), blk.q.data_ptr(), m, m)
            self._gram(NEW_arr, m, 1, m, self.r.data_ptr(), 1, 1, self.alpha.data_ptr(), tag="gram_vec")
        finish_now = (k % self.every != 0)
        xr_fused = fused and m <= 16
        if xr_fused:
            self._ensure_history(k + 1)
            self._timed("spmm_xr", lambda: _lib.call(
                "ekcg_stencil_xr", self.op.desc_ref(), blk.q.data_ptr(), m, WA, m, m,
                self.alpha.data_ptr(), self.x.data_ptr(), self.r.data_ptr(), part.data_ptr(),
                self.counter.data_ptr(), live, self._karg(k), self.kmax, self.stag_window, self.history.data_ptr(),
                1 if finish_now else 0, self.rho2.data_ptr(), st))
        else:
            self._apply_op(blk.q.data_ptr(), m, WA, m, m)  # A W_k -> WA: next candidate
            self._timed("xr_update", lambda: _lib.call(
                "ekcg_xr_update", blk.q.data_ptr(), m, WA, m, self.alpha.data_ptr(), m,
                self.x.data_ptr(), self.r.data_ptr(), n, self.vpart.data_ptr(), live, st))
            _lib.call("ekcg_reduce", self.vpart.data_ptr(), self.vchunks, 1, self.rho2.data_ptr(), live, st)
        self._append(blk)
        if not finish_now:
            slot = k // self.every - 1
            self._ensure_checks(slot + 1)
            self._residual_sq(self.x, self.tr2, live)
            _lib.call("ekcg_store_norm", self.tr2.data_ptr(), self.checks.data_ptr(), slot, live, st)
        if not (xr_fused and finish_now):
            self._ensure_history(k + 1)
            _lib.call("ekcg_finish", self.ctrl.data_ptr(), self.rho2.data_ptr(), self._karg(k), self.kmax, self.stag_window,
                      self.history.data_ptr(), st)
        self._account(k, d, m, fresh, t)

    def _candidate_split(self, WA, t, m):
        """split(r) (partition.py:48-55), preconditioned as in solvers.py:331-336:
        M^-1 split(r) when the factor blocks align with the subdomains, else
        L^-T split(L^-1 r)."""
        n, st, live = self.n, self.stream, self.live
        owner = self.owner_dev.data_ptr()
        pc = self.pc
        if pc is None:
            _lib.call("ekcg_split", self.r.data_ptr(), owner, WA, n, t, m, live, st)
        elif self.pc_aligned:
            _lib.call("ekcg_split", self.r.data_ptr(), owner, WA, n, t, m, live, st)
            self._minv(WA, m, WA, m, t)
        else:
            pc.apply(pc.FORWARD, self.r.data_ptr(), 1, self.tmpv2.data_ptr(), 1, 1, live, st)
            _lib.call("ekcg_split", self.tmpv2.data_ptr(), owner, WA, n, t, m, live, st)
            pc.apply(pc.BACKWARD, WA, m, self.WC.data_ptr(), m, t, live, st)
            _lib.call("ekcg_copy_cols", self.WC.data_ptr(), m, WA, m, n, t, live, st)

    def _normed(self, v, live):
        """Pointer to the vector whose 2-norm is the residual norm: v, or L v in explicit-hat mode."""
        if self.norm_pc is None:
            return v.data_ptr()
        pc = self.norm_pc
        pc.apply(pc.MULT_L, v.data_ptr(), 1, self.tmpv3.data_ptr(), 1, 1, live, self.stream)
        return self.tmpv3.data_ptr()

    def _minv(self, X, ldx, Y, ldy, w):
        """Y = M^-1 X = L^-T L^-1 X (blockjacobi.py:155-157) through the scratch block WC."""
        pc, st, live = self.pc, self.stream, self.live
        scratch = self.WC.data_ptr() if w > 1 else self.tmpv3.data_ptr()
        pc.apply(pc.FORWARD, X, ldx, scratch, w, w, live, st)
        pc.apply(pc.BACKWARD, scratch, w, Y, ldy, w, live, st)

    def _chain(self, V, m, t):
        """s-step chain V^(i+1) = A V^(i) on column slabs of width t (s-step)."""
        for i in range(1, self.s):
            self._apply_op(V + F64 * (i - 1) * t, m, V + F64 * i * t, m, t, tag="spmm_chain")

    def _residual_sq(self, x, out, live):
        """out = |b - A x|^2 (solvers.py:342,401)."""
        self._apply_op(x.data_ptr(), 1, self.tmpv.data_ptr(), 1, 1, tag="spmv", live=live)
        _lib.call("ekcg_sub", self.b.data_ptr(), self.tmpv.data_ptr(), self.tmpv.data_ptr(), self.n, live,
                  self.stream)
        _lib.call("ekcg_sumsq", self._normed(self.tmpv, live), self.n, self.vpart.data_ptr(), live, self.stream)
        _lib.call("ekcg_reduce", self.vpart.data_ptr(), self.vchunks, 1, out.data_ptr(), live, self.stream)

    def _ensure_history(self, length):
        if self.history.numel() < length:
            new = torch.zeros(max(length, 2 * self.history.numel()), dtype=torch.float64, device=self.device)
            new[: self.history.numel()].copy_(self.history)
            self.history = new

    def _ensure_checks(self, length):
        if self.checks.numel() < length:
            new = torch.zeros(max(length, 2 * self.checks.numel()), dtype=torch.float64, device=self.device)
            new[: self.checks.numel()].copy_(self.checks)
            self.checks = new

    def _account(self, k, d, m, fresh, t):
        """Record (k, d, m) for the traffic/flop model and peak replay."""
        self.launch_k.append((k, d, m))

    def _nnz(self):
        op = self.op
        while getattr(op, "nnz", None) is None and hasattr(op, "op"):  # composite (explicit-hat) operator
            op = op.op
        if getattr(op, "nnz", None) is not None:
            return op.nnz
        shape = op.shape
        tot = self.n
        for ax in range(len(shape)):
            other = self.n // shape[ax]
            tot += 2 * (shape[ax] - 1) * other
        return tot

    # -------------------------------------------------------------- control
    def _read_ctrl(self):
        self.ctrl_host.copy_(self.ctrl, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        raw = self.ctrl_host.numpy()
        ints = raw[:32].view(np.int32)
        dbl = raw[32:80].view(np.float64)
        return {
            "live": int(ints[0]), "status": int(ints[1]), "k_done": int(ints[2]), "brk_kind": int(ints[3]),
            "brk_col": int(ints[4]), "brk_iter": int(ints[5]), "brk_pivot": float(dbl[0]),
            "brk_scale": float(dbl[1]), "rho0": float(dbl[2]), "tol_abs": float(dbl[3]),
            "last_rho": float(dbl[5]),
        }

    def _snapshot(self, j):
        buf = self.snap_bufs[j % len(self.snap_bufs)]
        buf.copy_(self.ctrl, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return buf, ev

    def _wait_snapshot(self, snap):
        buf, ev = snap
        ev.synchronize()
        raw = buf.numpy()
        ints = raw[:32].view(np.int32)
        dbl = raw[32:80].view(np.float64)
        return {"live": int(ints[0]), "status": int(ints[1]), "k_done": int(ints[2]),
                "tol_abs": float(dbl[3]), "last_rho": float(dbl[5])}

    @staticmethod
    def _batch_size(lookahead, seen, k_next):
        """Iterations to queue next: the doubling look-ahead, cut to what the residual
        decay between the last two snapshots predicts is still needed (x1.25 + 2), so
        that few gated no-op iterations sit in the queue past convergence.  Never 0;
        a low prediction only costs an extra poll.  Identical on every row shard
        (the snapshots hold allreduced values)."""
        if len(seen) < 2:
            return lookahead
        (k0, r0), (k1, r1) = ((c["k_done"], c["last_rho"]) for c in seen[-2:])
        tol_abs = seen[-1]["tol_abs"]
        if k1 <= k0 or not (0.0 < r1 < r0) or not tol_abs > 0.0:
            return lookahead
        left = math.log(tol_abs / r1) / math.log(r1 / r0) * (k1 - k0) if r1 > tol_abs else 0.0
        need = math.ceil(1.25 * left) + 2 - ((k_next - 1) - k1)
        return max(1, min(lookahead, need))

    # ---------------------------------------------------------------- solve
    def solve(self, b, x0=None, x_star=None, on_iteration=None, numpy_io=None):
        """numpy_io: return x (and callback states) as numpy (default: when b is not a tensor)."""
        cfg = self.cfg
        dev = self.device
        numpy_io = (not isinstance(b, torch.Tensor)) if numpy_io is None else numpy_io
        self._setup()
        t_wall0 = time.perf_counter()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        self._begin(b, x0)

        sync_each = (on_iteration is not None or self.retention == "restart-tol"
                     or cfg.switch_tol is not None or self.sync_mode)
        if not sync_each and self._cluster_eligible():
            ctrl = self._solve_cluster()
            ev1.record()
            ev1.synchronize()
            solve_s = ev0.elapsed_time(ev1) / 1e3
            return self._report(ctrl, x_star, numpy_io, solve_s, time.perf_counter() - t_wall0)
        host_hist = None
        if sync_each:
            c = self._read_ctrl()
            host_hist = [c["rho0"]]
        k = 1
        lookahead = batch = 1
        seen = []
        tol1 = 1.0
        ctrl = None
        snaps = []
        graphs = {} if (not sync_each and self._graph_eligible()) else None
        self._graphs = graphs
        while k <= self.kmax:
            if sync_each:
                self._enqueue(k, tol1)
                ctrl = self._read_ctrl()
                if ctrl["k_done"] == k:
                    rho = ctrl["last_rho"]
                    tol1 = abs(rho - host_hist[-1]) / host_hist[0]
                    host_hist.append(rho)
                    if on_iteration is not None:
                        on_iteration(self._state(k, rho, tol1, numpy_io))
                if ctrl["live"] == 0:
                    break
                k += 1
            else:
                # run ahead: snapshot the control block after every batch and
                # only wait for the PREVIOUS batch's snapshot, so the GPU queue
                # never drains while the host polls
                for _ in range(batch):
                    if k > self.kmax:
                        break
                    w = self.window
                    if (graphs is not None and k > 2 * w and k % self.every != 0
                            and len(self.retained) == w):
                        phase = (k - 1) % w
                        g = graphs.get(phase)
                        if g is None:  # first visit of this phase in steady state: capture
                            g = graphs[phase] = self._capture_iteration(k)
                        else:
                            self._host_step(k)
                        g.replay()
                    else:
                        self._enqueue(k, 1.0)
                    k += 1
                snaps.append(self._snapshot(len(snaps)))
                if len(snaps) >= 2:
                    prev = self._wait_snapshot(snaps[-2])
                    if prev["live"] == 0:
                        break
                    seen.append(prev)
                lookahead = min(2 * lookahead, self.max_lookahead)
                batch = self._batch_size(lookahead, seen, k) if self.predict_batches else lookahead
        ctrl = self._read_ctrl()  # after a full sync: the final state
        ev1.record()
        ev1.synchronize()
        solve_s = ev0.elapsed_time(ev1) / 1e3
        return self._report(ctrl, x_star, numpy_io, solve_s, time.perf_counter() - t_wall0)

    # -------------------------------------------------------- cluster solve
    def _cluster_eligible(self):
        """The one-kernel cluster solve (csrc/cluster_solve.cu) covers unpreconditioned SRE-CG /
        SRE-CG2 with a truncation window, s = 1, t <= 16, window <= 4 (t <= 8) or 2 (t = 16), on a whole-grid
        stencil operator or a CSR matrix with rows of at most 8 entries."""
        from .operators import CsrOperator, StencilOperator
        if not self.cluster_ok or self.use_cluster is False or self.kernel_timer is not None or self.no_fuse:
            return False
        if (self.method not in ("sre-cg2", "sre-cg") or self.s != 1 or self.retention != "trunc"
                or self.pc is not None or self.norm_pc is not None or self.cfg.switch_tol is not None
                or self.lean or self.window is None or self.kmax + 1 > self.history.numel()):
            return False
        t = self.t_cur
        if not _lib.query("ekcg_cluster_solve_fits", self.n, t, self.window):
            return False
        # measured crossover against the launch-per-phase engine (tools/cluster_time.py): t = 8 wins up to
        # n t ~ 2.3e5 (n = 25,600: 88 vs 94 us per iteration; n = 32,761: 106 vs 100), t = 16 (8-CTA
        # cluster) up to n t ~ 1.3e5
        if self.use_cluster == "auto" and self.n * t > (200_000 if t <= 8 else 131_072):
            return False
        op = self.op
        if isinstance(op, StencilOperator):
            return True
        if isinstance(op, CsrOperator):
            if not hasattr(op, "_max_row"):
                op._max_row = int((op.row_ptr[1:] - op.row_ptr[:-1]).max().item()) if self.n else 0
            return op._max_row <= 8
        return False

    def _solve_cluster(self):
        """Run the whole solve in the cluster kernel; returns the final control block."""
        from .operators import StencilOperator
        n, t, w = self.n, self.t_cur, self.window
        span = self._span(n * t)
        blocks = torch.empty((2 * w + 3) * span + self._span(n), dtype=torch.float64, device=self.device)
        nchk = max(1, self.kmax // self.every + 1)
        self._ensure_checks(nchk)
        op = self.op
        if isinstance(op, StencilOperator):
            desc, rp, ci, vv = op.desc_ref(), None, None, None
        else:
            desc, rp, ci, vv = None, op.row_ptr.data_ptr(), op.col_idx.data_ptr(), op.values.data_ptr()
        _lib.call("ekcg_cluster_solve", desc, rp, ci, vv, n, t, w, self.kmax, self.every,
                  self.owner_dev.data_ptr(), self.b.data_ptr(), self.x.data_ptr(), self.r.data_ptr(),
                  blocks.data_ptr(), span, self.ctrl.data_ptr(), self.history.data_ptr(), self.checks.data_ptr(),
                  1e-14, None if self.cluster_ticks is None else self.cluster_ticks.data_ptr(), self.stream)
        ctrl = self._read_ctrl()
        if ctrl["status"] == 5:
            raise _lib.KernelError("ekcg_cluster_solve refused the matrix: a CSR row holds more than 8 entries")
        self._cluster_blocks = blocks
        self.ran_cluster = True
        last = ctrl["k_done"] + (1 if ctrl["status"] == 3 else 0)
        self.launch_k = [(k, min(k - 1, w), t) for k in range(1, last + 1)]
        return ctrl

    def _begin(self, b, x0):
        """Upload b / x0, r = b - A x, rho0 = |r| and the control block (solvers.py:341-345)."""
        dev, st = self.device, self.stream
        self.b = torch.as_tensor(b, dtype=torch.float64).to(dev, non_blocking=False).contiguous()
        if x0 is None:
            self.x = torch.zeros(self.n, dtype=torch.float64, device=dev)
        else:
            self.x = torch.as_tensor(x0, dtype=torch.float64).to(dev).clone().contiguous()
        self.r = torch.empty(self.n, dtype=torch.float64, device=dev)
        self._apply_op(self.x.data_ptr(), 1, self.tmpv.data_ptr(), 1, 1, tag="spmv", live=None)
        _lib.call("ekcg_sub", self.b.data_ptr(), self.tmpv.data_ptr(), self.r.data_ptr(), self.n, None, st)
        _lib.call("ekcg_sumsq", self._normed(self.r, None), self.n, self.vpart.data_ptr(), None, st)
        _lib.call("ekcg_reduce", self.vpart.data_ptr(), self.vchunks, 1, self.rho2.data_ptr(), None, st)
        self._allreduce(self.rho2)
        _lib.call("ekcg_start", self.ctrl.data_ptr(), self.rho2.data_ptr(), self.tol, self.history.data_ptr(), st)

    def _allreduce(self, t):
        """Sum a small partial across row shards (no-op on one GPU)."""

    def _final_metrics(self, x_star):
        """(|b - A x|, |x - x*| / |x*|) of the final iterate (solvers.py:289-291)."""
        self._residual_sq(self.x, self.tr2, None)
        true_res = float(torch.sqrt(self.tr2).item())
        rel = None
        if x_star is not None:
            xs = torch.as_tensor(x_star, dtype=torch.float64).to(self.device)
            rel = float((torch.linalg.vector_norm(self.x - xs) / torch.linalg.vector_norm(xs)).item())
        return true_res, rel

    def _output_x(self, numpy_io):
        if not numpy_io:
            return self.x
        # into pinned host memory: torch's host caching allocator hands a freed result's pages to the next
        # call, so a repeated 537 MB readback takes ~10 ms instead of ~250 ms of pageable page faults
        out = torch.empty(self.x.numel(), dtype=torch.float64, pin_memory=True)
        out.copy_(self.x)
        return out.numpy()

    def _state(self, k, rho, tol1, numpy_io):
        conv = (lambda t: t.cpu().numpy()) if numpy_io else (lambda t: t.clone())
        blocks = []
        for b in self.retained:
            q = b.q[: self.n * b.width].view(self.n, b.width)
            if b.aq is not None:
                aq = b.aq[: self.n * b.width].view(self.n, b.width)
            else:  # lean scheme: materialise A Q for the callback only
                aq = torch.empty_like(q)
                self._apply_op(q.data_ptr(), b.width, aq.data_ptr(), b.width, b.width, tag="spmm", live=None)
            blocks.append((q, aq))
        return {"k": k, "x": conv(self.x), "r": conv(self.r), "rho": rho, "tol1": tol1,
                "store": BasisStore(self.window, blocks, self.peak, to_host=numpy_io),
                "partition": self.part_obj}

    def _report(self, ctrl, x_star, numpy_io, solve_s, wall_s):
        status_code = ctrl["status"]
        k_done = ctrl["k_done"]
        status = _STATUS.get(status_code)
        if status is None:
            # loop exhausted kmax without the device flag (cannot happen) or rho0 == 0
            status = "converged" if ctrl["last_rho"] <= ctrl["tol_abs"] else "maxiter"
        notes = list(self.notes_init)
        if status_code == 3:
            if ctrl["brk_kind"] == 1:
                msg = f"zero column {ctrl['brk_col']} entering Pre-CholQR"
            else:
                msg = f"pivot {ctrl['brk_pivot']:.3e} at column {ctrl['brk_col']} (scale {ctrl['brk_scale']:.3e})"
            notes.append(f"basis breakdown at iteration {ctrl['brk_iter']}: {msg}")
        elif status_code == 4:
            notes.append(f"no residual decrease over {self.stag_window} iterations")
        history = self.history[: k_done + 1].cpu().numpy().copy()
        last_attempted = k_done + 1 if status_code == 3 else k_done
        # host bookkeeping ran ahead: replay the store model up to the real stop
        restarts = [r for r in self.restarts if r <= last_attempted]
        switch_it = self.switch_iteration if (self.switch_iteration or 0) <= last_attempted else None
        peak = self._replay_peak(k_done)
        nchecks = k_done // self.every
        checks_v = self.checks[:nchecks].cpu().numpy() if nchecks else np.zeros(0)
        checks = [((i + 1) * self.every, float(checks_v[i])) for i in range(nchecks)]
        true_res, rel = self._final_metrics(x_star)
        x_out = self._output_x(numpy_io)
        model_bytes = sum(self._iter_bytes(d, m) for kk, d, m in self.launch_k if kk <= k_done)
        model_flops = sum(self._iter_flops(d, m) for kk, d, m in self.launch_k if kk <= k_done)
        rep = ConvergenceReport(
            status=status, iterations=len(history) - 1, residual_history=history,
            switch_iteration=switch_it, restart_iterations=restarts, peak_block_vectors=peak,
            relative_error=rel, true_residual=true_res, true_residual_checks=checks, x=x_out, notes=notes,
            solve_seconds=solve_s, iterations_per_second=(k_done / solve_s if solve_s > 0 else None),
            model_bytes=model_bytes, model_flops=model_flops)
        rep.wall_seconds = wall_s
        return x_out, rep

    def _iter_bytes(self, d, m):
        """8[(4d + 11) n m + 5 n] + 2 M_A, plus the s-step chain
        (s - 1)(16 n t + M_A) when s > 1."""
        n = self.n
        t = m // self.s
        chain = (self.s - 1) * (16.0 * n * t + self.op.matrix_bytes())
        return 8.0 * ((4 * d + 11) * n * m + 5 * n) + 2 * self.op.matrix_bytes() + chain

    def _iter_flops(self, d, m):
        n = self.n
        t = m // self.s
        chain = (self.s - 1) * 2.0 * self._nnz() * t
        return (8 * d + 6) * m * m * n + 4.0 * self._nnz() * m + 6.0 * m * n + chain

    def _replay_peak(self, k_done):
        """peak_block_vectors with append-before-trim (solvers.py:163-170) over completed iterations."""
        cols, peak, blocks = 0, 0, []
        restarts = set(self.restarts)
        for kk, d, m in self.launch_k:
            if kk > k_done:
                break
            if kk in restarts:
                blocks, cols = [], 0
            blocks.append(m)
            cols += m
            peak = max(peak, cols)
            if self.window is not None:
                while len(blocks) > self.window:
                    cols -= blocks.pop(0)
        return peak
