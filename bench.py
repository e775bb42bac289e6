"""Benchmark: enlarged-CG iterations/s on B200 (BASELINE.json metric), one JSON line.

Default workload = BASELINE config 5 at full size, the largest configuration
that fits one B200 (truncated SRE-CG2, t=64, trunc 3, heterogeneous 2D
5-point diffusion on 8192^2 with 16x16-cell log-uniform tiles, 8x8 boxes,
b ~ U(-1,1) seed 5), run in the lean scheme (w + 2 = 5 blocks of 34.4 GB).
One "step" is a fixed window of K = 8 iterations from x0 = 0 (kmax = 8; the
retained history fills to d = 3 at iteration 4); value = iterations / device
time with the inputs resident in HBM.  Config 5 converges in thousands of
iterations (tol 1e-6), so a whole solve is not a benchmark step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--edge E] [--window K]
  python bench.py --impl reference ...   # the reference algorithm on the host CPU (oracle port)

`--config 2` gives the round-1 workload (one complete config-2 solve per step).
Under torchrun (N > 1) the rows are sharded across the ranks (one solve,
strong scaling: halo exchange + NCCL allreduce, paper_2305_19013_b200/sharded.py);
timing is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
import types
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "enlarged-CG iterations/s + HBM GB/s vs roofline at 1/2/4/8 B200"
UNIT = "iterations/s"
# fixed iteration window per step, per config (None = one complete solve)
WINDOW = {1: None, 2: None, 3: 16, 4: 6, 5: 8}
# CPU-sample instance edge per config (reference arm / cpu_baseline): the same generator, partition
# and seeds on a row-scaled instance, its rate scaled by n_sample / n_full (row-linear work)
CPU_EDGE = {1: None, 2: None, 3: 32, 4: 64, 5: 256}
F64_PEAK_FILE = ROOT / "profiles" / "fp64_peak.json"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--edge", type=int, default=None)
    ap.add_argument("--window", type=int, default=None, help="iterations per step (default per config)")
    ap.add_argument("--form", default="stencil", choices=["stencil", "csr"])
    ap.add_argument("--e2e-form", default="stencil", choices=["stencil", "csr"],
                    help="operator handed to enlarged_solve in the e2e leg (host field or host CSR)")
    ap.add_argument("--cpu-iters", type=int, default=None, help="iterations in the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-kernel-timer", action="store_true", help="skip the per-kernel CUDA events")
    ap.add_argument("--no-grid-detect", action="store_true",
                    help="keep CSR matrices on the CSR kernels (no grid-pattern detection)")
    ap.add_argument("--kernel-timer-small", action="store_true",
                    help="config 1: time the launch-per-phase engine per kernel instead of the one-kernel cluster solve")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def peaks():
    """(HBM GB/s, source), (FP64 TFLOP/s, source)."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        hbm = (float(json.loads(p.read_text())["hbm_gbs"]), "measured: MEASURED_PEAKS.json hbm_gbs")
    else:
        hbm = (6650.0, "fallback: B200_PROFILING.md")
    if F64_PEAK_FILE.exists():
        d = json.loads(F64_PEAK_FILE.read_text())
        fp = (float(d["dmma_tflops"]), f"measured by this repo: {d['source']}")
    else:
        fp = (37.1, "builder-measured DMMA.8x8x4 peak (profiles/r01_fp64_peak.txt)")
    return hbm, fp


# ---------------------------------------------------------------------------
# clocks sampler (NVML during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock and throttle reasons sampled with NVML from a background thread
    during the timed region (every 100 ms; NVML calls release the GIL).  An
    `nvidia-smi -lms` child at 100 ms was measured to slow kernel launches."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index, interval=0.1):
        self.index = index
        self.interval = interval
        self.samples = []
        self.stop_evt = threading.Event()
        self.thread = None
        self.ok = False

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        nv = self.nvml
        while not self.stop_evt.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.handle)
                self.samples.append((mhz, rs))
            except Exception:
                pass
            self.stop_evt.wait(self.interval)

    def stop(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self.stop_evt.set()
        self.thread.join(2)
        reasons = set()
        for _, rs in self.samples:
            for name, bit in self.REASONS.items():
                if rs & bit:
                    reasons.add(name)
        mhz = [s[0] for s in self.samples]
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(mhz), "source": "nvml"}


# ---------------------------------------------------------------------------
# CPU legs (oracle port of the reference algorithm)
# ---------------------------------------------------------------------------
def cpu_problem(config, edge):
    """The instance the CPU legs run: the full config where the host holds it (1, 2),
    otherwise the same generator on CPU_EDGE rows (configs 3-5)."""
    from paper_2305_19013_b200.problems import FULL_EDGE, make_config
    e = edge if edge is not None else (CPU_EDGE.get(config) or FULL_EDGE[config])
    return make_config(config, e, device_rhs=False)


def cpu_sample(prob, iters):
    from oracle import ekcg_oracle as orc
    A = prob.csr()
    kw = dict(prob.solver_kwargs)
    t = kw.pop("t")
    kw["kmax"] = iters
    t0 = time.perf_counter()
    out = orc.run_oracle(A.row_ptr, A.col_idx, A.values, prob.b, prob.partition.owner(), t, **kw)
    dt = time.perf_counter() - t0
    return out["iterations"], dt


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


def cpu_iters(args):
    if args.cpu_iters:
        return args.cpu_iters
    w = args.window if args.window is not None else WINDOW.get(args.config)
    return w if w is not None else {1: 130, 2: 12}.get(args.config, 5)


def cpu_leg(args, n_full, samples):
    """it/s of the reference algorithm at the benchmarked config (rate scaled by rows)."""
    prob = cpu_problem(args.config, None if args.edge is None else args.edge)
    iters = cpu_iters(args)
    tot_it, tot_s = 0, 0.0
    for _ in range(samples):
        it, dt = cpu_sample(prob, iters)
        tot_it += it
        tot_s += dt
    scale = prob.n / n_full
    value = tot_it / tot_s * scale
    if prob.n == n_full:
        what = f"first {iters} iterations of {prob.name}"
    else:
        what = (f"first {iters} iterations of {prob.name} ({prob.n} of {n_full} rows; same generator, partition "
                f"and seeds), {tot_it / tot_s:.3f} it/s there, scaled by n_sample / n_full = {scale:.3g}")
    return value, (f"{what}; reference algorithm (numpy/OpenBLAS oracle port, bitwise the reference at "
                   f"golden sizes), {samples} sample(s), {tot_s:.1f} s")


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2305_19013_b200.problems import FULL_EDGE
    full_edge = args.edge or FULL_EDGE[args.config]
    n_full = full_edge ** (2 if args.config in (1, 5) else 3)
    prob = cpu_problem(args.config, None if args.edge is None else args.edge)
    iters = cpu_iters(args)
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_sample(prob, min(iters, 2))
    value, sample = cpu_leg(args, n_full, args.steps)
    window = args.window if args.window is not None else WINDOW.get(args.config)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * (window or iters) / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": _workload_name(args.config, args.edge),
                   "n": n_full, "t": prob.solver_kwargs["t"], "s": prob.solver_kwargs.get("s", 1),
                   "iterations_per_step": window, "sample_edge": prob.edge},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def _workload_name(config, edge):
    from paper_2305_19013_b200.problems import CONFIG_NAMES, FULL_EDGE
    e = edge or FULL_EDGE[config]
    name = CONFIG_NAMES[config] if e == FULL_EDGE[config] else f"{CONFIG_NAMES[config]}@{e}"
    w = WINDOW.get(config)
    return name if w is None else f"{name}, {w}-iteration window from x0=0"


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------
def tag_model(tag, n, m, d, nnz, mat_bytes):
    """(algorithmic bytes, flops) of one tagged launch."""
    nm = float(n) * m
    if tag == "hist_gram":      # [AQ_1..AQ_d]^T W (or Q^T (A W) in the lean scheme)
        return 8.0 * (d + 1) * nm, 2.0 * d * m * nm
    if tag == "hist_update":    # W - sum Q_i C_i
        return 8.0 * (d + 2) * nm, 2.0 * d * m * nm
    if tag == "gram_self":      # W^T W (one block read; symmetric: m (m + 1) / 2 distinct entries)
        return 8.0 * nm, (m + 1.0) * nm
    if tag == "gram_aw":        # W0^T (A W0)
        return 16.0 * nm, 2.0 * m * nm
    if tag in ("spmm", "spmm_proj", "spmm_chain"):
        return 16.0 * nm + mat_bytes, 2.0 * nnz * m
    if tag == "tri_apply":      # W S, S upper triangular
        return 16.0 * nm, 1.0 * m * nm
    if tag == "xr_update":      # x += W alpha, r -= AW alpha, |r|^2
        return 8.0 * (2 * nm + 4 * n), 4.0 * nm
    if tag == "gram_vec":       # W^T r
        return 8.0 * (nm + n), 2.0 * nm
    return None


TIMED_TAGS = ("hist_gram", "hist_update", "gram_self", "gram_aw", "spmm", "spmm_proj", "spmm_chain", "tri_apply",
              "xr_update", "gram_vec")


class KernelTimer:
    """CUDA-event timing of tagged launches on the launching stream.

    Only launches with d >= d_min retained blocks are bracketed (config 2: the
    GPU-bound late iterations, so the host cost of the event records hides
    behind device work); events come from a pool created up front and are
    harvested after each step's final sync.  Each record keeps (tag, k, d, m).
    """

    def __init__(self, torch, tags, d_min=0, pool=8192):
        self.torch = torch
        self.tags = set(tags)
        self.d_min = d_min
        self.pool = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                     for _ in range(pool)]
        self.used = []
        self.records = []  # (tag, k, d, m, ms)
        self.enabled = False
        self.engine = None

    def __call__(self, tag, fn):
        cur = getattr(self.engine, "_cur", None)
        if (not self.enabled or tag not in self.tags or cur is None or cur[1] < self.d_min
                or len(self.used) >= len(self.pool)):
            fn()
            return
        e0, e1 = self.pool[len(self.used)]
        e0.record()
        fn()
        e1.record()
        k, d, m = cur
        if tag == "spmm_chain":  # the s-step chain applies A to one t-column slab of the s t-wide block
            m //= max(1, int(getattr(self.engine, "s", 1)))
        self.used.append((tag, k, d, m))

    def harvest(self, k_done):
        """Call after a full device sync; drops launches past the stopping iteration."""
        for (tag, k, d, m), (e0, e1) in zip(self.used, self.pool):
            if k <= k_done:
                self.records.append((tag, k, d, m, e0.elapsed_time(e1)))
        self.used = []


def roofline_block(timer, n, nnz, mat_bytes, hbm, fp64, traffic_db, workload):
    per_tag = {}
    for tag, k, d, mm, ms in timer.records:
        model = tag_model(tag, n, mm, d, nnz, mat_bytes)
        if model is None:
            continue
        acc = per_tag.setdefault(tag, [0.0, 0.0, 0.0, 0, []])
        acc[0] += model[0]
        acc[1] += model[1]
        acc[2] += ms
        acc[3] += 1
        acc[4].append(d)
    if not per_tag:
        return None
    tot_ms = sum(v[2] for v in per_tag.values())
    dom = max(per_tag, key=lambda t: per_tag[t][2])
    b, f, ms, cnt, ds = per_tag[dom]
    s = ms / 1e3
    t_hbm, t_fp = b / (hbm[0] * 1e9), f / (fp64[0] * 1e12)
    bound = "fp64" if t_fp > t_hbm else "hbm"
    if bound == "fp64":
        achieved, peak, unit, psrc = f / s / 1e12, fp64[0], "TFLOP/s", fp64[1]
    else:
        achieved, peak, unit, psrc = b / s / 1e9, hbm[0], "GB/s", hbm[1]
    tr = traffic_db.get(f"{workload}|{dom}") if traffic_db else None
    out = {
        "bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
        "traffic": tr["dram_bytes_per_launch"] if tr else None,
        "kernel": dom, "kernel_share_of_timed": ms / tot_ms, "launches": cnt,
        "alg_bytes_per_launch": b / cnt, "alg_flops_per_launch": f / cnt, "avg_launch_ms": ms / cnt,
        "hbm_frac": (b / s / 1e9) / hbm[0], "fp64_frac": (f / s / 1e12) / fp64[0],
        "peak_source": psrc, "other_peak": {"hbm_gbs": hbm[0], "hbm_source": hbm[1], "fp64_tflops": fp64[0],
                                            "fp64_source": fp64[1]},
        "per_kernel": {t: {"GBs": v[0] / (v[2] / 1e3) / 1e9, "TFLOPs": v[1] / (v[2] / 1e3) / 1e12,
                           "ms_total": round(v[2], 3), "launches": v[3],
                           "roof_frac": max(v[0] / (hbm[0] * 1e9), v[1] / (fp64[0] * 1e12)) / (v[2] / 1e3)}
                       for t, v in per_tag.items()},
        "timed_launches": f"tagged launches with d >= {timer.d_min} retained blocks, all timed steps",
    }
    if tr:
        out["traffic_source"] = tr.get("source")
        out["traffic_alg_bytes"] = tr.get("alg_bytes")
        out["traffic_d"] = tr.get("d")
    return out


def run_ours(args):
    # one engine's blocks are freed before the next step allocates its own; expandable segments keep
    # the 34 GB config-5 blocks from fragmenting the caching allocator across steps
    os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    import paper_2305_19013_b200 as pk
    from paper_2305_19013_b200 import _lib
    from paper_2305_19013_b200.engine import DeviceEngine
    from paper_2305_19013_b200.problems import make_config
    from paper_2305_19013_b200.sharded import ShardedEngine

    window = args.window if args.window is not None else WINDOW.get(args.config)
    prob = make_config(args.config, args.edge)
    kw = dict(prob.solver_kwargs)
    if window is not None:
        kw["kmax"] = window
    cfg = pk.SolverConfig(**kw)
    if args.no_grid_detect:
        from paper_2305_19013_b200 import operators as _ops
        _ops.DETECT_GRID = False
    # --form csr: the operator the reference-facing call builds from a CSR matrix (grid patterns are detected
    # and applied in stencil form unless --no-grid-detect)
    op = prob.stencil(dev) if args.form == "stencil" else pk.as_operator(prob.csr(), dev)
    b_dev = torch.as_tensor(prob.b, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)  # 256 MB > L2 (126 MB)
    timer = KernelTimer(torch, TIMED_TAGS, d_min=16 if args.config == 2 else 0)
    sharded = world > 1
    workload = _workload_name(args.config, args.edge)

    def solve_once(timed):
        eng = (ShardedEngine if sharded else DeviceEngine)(op, prob.partition, cfg, device=dev)
        # per-kernel events need one launch per phase; small truncated-window problems (config 1) run as ONE
        # cluster kernel unless --kernel-timer-small asks for the launch-per-phase engine's breakdown
        if not (args.config == 1 and not args.kernel_timer_small):
            eng.kernel_timer = timer
        timer.engine = eng
        timer.enabled = timed and not args.no_kernel_timer
        x, rep = eng.solve(b_dev)
        timer.engine = None  # the timer must not keep a finished solve's blocks alive
        return rep, eng

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        solve_once(False)
    barrier()

    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _lib.query("ekcg_launch_count")
    step_ms, iters, reps = [], 0, []
    n_rows, lean, ran_cluster = prob.n, None, False
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush between timed steps (outside the events)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep, eng = solve_once(True)
        e1.record()
        e1.synchronize()
        timer.harvest(rep.iterations)
        step_ms.append(e0.elapsed_time(e1))
        iters += rep.iterations
        rep.x = None  # the solution stays with its engine, which is released below
        reps.append(rep)
        n_rows, lean = eng.n, eng.lean  # local rows on a shard
        ran_cluster = bool(getattr(eng, "ran_cluster", False))
        nnz, mat_bytes = eng._nnz(), eng.op.matrix_bytes()
        eng = None  # release the solve's blocks before the next step allocates its own
    barrier()
    launches = _lib.query("ekcg_launch_count") - launches0
    clk = clocks.stop()
    if rank == 0:
        print(f"[bench] step ms: {[round(v, 2) for v in step_ms]}", file=sys.stderr)

    tot_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    value = iters / (tot_ms / 1e3)  # sharded: every rank iterates the same solve

    hbm, fp64 = peaks()
    traffic_db = {}
    tpath = ROOT / "profiles" / "r02_traffic.json"
    if tpath.exists():
        traffic_db = json.loads(tpath.read_text())
    roofline = roofline_block(timer, n_rows, nnz if not sharded else nnz // world, mat_bytes, hbm, fp64,
                              traffic_db, workload)
    model_bytes = sum(r.model_bytes for r in reps)
    model_flops = sum(r.model_flops for r in reps)
    if roofline is None and ran_cluster:
        # one kernel per solve: the SURVEY 8(d) traffic model of the whole solve against HBM.  The blocks
        # are L2-resident and the kernel is latency-bound, so the fraction is small.
        s_tot = tot_ms / 1e3
        roofline = {"bound": "hbm", "achieved": model_bytes / s_tot / 1e9, "peak": hbm[0], "unit": "GB/s",
                    "frac": model_bytes / s_tot / 1e9 / hbm[0], "traffic": None,
                    "kernel": "cluster_solve_kernel (the whole solve in one kernel; L2-resident, latency-bound)",
                    "peak_source": hbm[1]}
    if roofline is not None:
        # whole-step model (per iteration max(bytes/HBM, flops/FP64), reference scheme)
        t_model = sum(max(r.model_bytes / (hbm[0] * 1e9), r.model_flops / (fp64[0] * 1e12)) for r in reps)
        roofline.update({
            "step_model_gbs": model_bytes / (tot_ms / 1e3) / 1e9,
            "step_model_tflops": model_flops / (tot_ms / 1e3) / 1e12,
            "step_model_frac": t_model / (tot_ms / 1e3),
            "step_model": "SURVEY 8(d): bytes 8[(4d+11)nm+5n]+2M_A, flops (8d+6)m^2n+4nnz m+6mn per iteration",
        })

    # ---- e2e through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        b_host = torch.from_numpy(np.ascontiguousarray(prob.b)).pin_memory()
        if args.e2e_form == "csr":
            # the reference-facing CSR object (SparseSpdMatrix layout): every call uploads the matrix
            csr = prob.csr()
            A_host = types.SimpleNamespace(n=csr.n, row_ptr=csr.row_ptr, col_idx=csr.col_idx, values=csr.values)
            mat_bytes_h2d = 8 * (csr.n + 1) + 12 * csr.nnz
            # a fresh host object per call: the operator cached on a matrix object would skip the upload
            make_A = lambda: types.SimpleNamespace(**vars(A_host))  # noqa: E731
            call = "enlarged_solve(host CSR matrix, host numpy b) -> host x, report"
        else:
            # the operator built from the host coefficient field inside the timed call (uploads the field)
            field = prob.kappa_field
            mat_bytes_h2d = 0 if field is None else int(np.asarray(field).nbytes)
            make_A = lambda: prob.stencil(dev)  # noqa: E731
            call = "enlarged_solve(StencilOperator(host kappa tile field), host numpy b) -> host x, report"
        pk.enlarged_solve(make_A(), b_host.numpy(), partition=prob.partition, cfg=cfg, device=dev)  # warm-up
        e2e_ms, e2e_it = [], 0
        for _ in range(max(1, args.steps)):
            flush.fill_(1.0)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            x, rep = pk.enlarged_solve(make_A(), b_host.numpy(), partition=prob.partition, cfg=cfg, device=dev)
            e1.record()
            e1.synchronize()
            e2e_ms.append(e0.elapsed_time(e1))
            e2e_it += rep.iterations
            x = None
        e2e_tot = sum(e2e_ms)
        if world > 1:
            t = torch.tensor([e2e_tot], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_tot = float(t.item())
        e2e = {"value": e2e_it / (e2e_tot / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * prob.n + mat_bytes_h2d,
               "d2h_bytes_per_step": 8 * prob.n + 8 * (reps[-1].iterations + 1), "call": call}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, sample = cpu_leg(args, prob.n, 1)
        cpu = {"value": v, "unit": UNIT, "cores": cores(), "kind": "port", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators of BASELINE.json's configs; no public dataset)",
            "config": {"workload": workload, "form": args.form, "n": prob.n, "t": prob.solver_kwargs["t"],
                       "s": prob.solver_kwargs.get("s", 1), "iterations_per_step": reps[-1].iterations,
                       "window": window, "status": reps[-1].status, "scheme": "lean" if lean else "cached A Q",
                       "parallelism": f"rows{world}" if sharded else "single",
                       "l2": "flushed (256 MB write) before every timed step; blocks of 8nm bytes >> L2",
                       "time_per_step_ms": tot_ms / args.steps},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
