"""Benchmark: enlarged-CG iterations/s on B200 (BASELINE.json metric), one JSON line.

Default workload = BASELINE config 2 (SRE-CG2, t=16, full history, 3D Poisson
64^3, box 4x2x2, b = A x*, x* ~ N(0,1) seed 1, tol 1e-8).  One "step" is one
complete solve to tol (111 iterations); value = iterations / device time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--edge E]
  python bench.py --impl reference ...   # the reference algorithm on the host CPU (oracle port)

Under torchrun (N > 1) the rows are sharded across the ranks (one solve,
strong scaling: halo exchange + NCCL allreduce, paper_2305_19013_b200/sharded.py);
timing is the max over ranks (stencil or CSR form).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--edge", type=int, default=None)
    ap.add_argument("--form", default="stencil", choices=["stencil", "csr"])
    ap.add_argument("--cpu-iters", type=int, default=None, help="iterations in the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-kernel-timer", action="store_true", help="skip the per-kernel CUDA events")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
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


def default_cpu_iters(config):
    return {1: 130, 2: 12, 3: 2, 4: 1, 5: 1}.get(config, 5)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2305_19013_b200.problems import make_config
    prob = make_config(args.config, args.edge, device_rhs=False)
    iters = args.cpu_iters or default_cpu_iters(args.config)
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_sample(prob, min(iters, 2))
    tot_it, tot_s = 0, 0.0
    for _ in range(args.steps):
        it, dt = cpu_sample(prob, iters)
        tot_it += it
        tot_s += dt
    value = tot_it / tot_s
    sample = (f"first {iters} iterations of {prob.name} (reference algorithm, numpy/OpenBLAS oracle port), "
              f"{args.steps} samples")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": prob.name, "n": prob.n, "t": prob.solver_kwargs["t"],
                   "iterations_per_step": iters},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------
class KernelTimer:
    """CUDA-event timing of the CGS2 history kernels on the launching stream.

    Only launches of the GPU-bound phase (d >= d_min retained blocks) are
    bracketed, so the host cost of the event records hides behind device work;
    events come from a pool created up front and are harvested after each
    step's final sync.  Each record keeps (tag, k, d, m) for the byte count.
    """

    def __init__(self, torch, tags, d_min=16, pool=4096):
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
        self.used.append((tag,) + tuple(cur))

    def harvest(self, k_done):
        """Call after a full device sync; drops launches past the stopping iteration."""
        for (tag, k, d, m), (e0, e1) in zip(self.used, self.pool):
            if k <= k_done:
                self.records.append((tag, k, d, m, e0.elapsed_time(e1)))
        self.used = []


def run_ours(args):
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

    prob = make_config(args.config, args.edge)
    cfg = pk.SolverConfig(**prob.solver_kwargs)
    op = prob.stencil(dev) if args.form == "stencil" else pk.CsrOperator(prob.csr(), dev)
    b_dev = torch.as_tensor(prob.b, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)  # 256 MB > L2 (126 MB)
    timer = KernelTimer(torch, ["hist_gram", "hist_update"])

    from paper_2305_19013_b200.sharded import ShardedEngine
    sharded = world > 1

    def solve_once(timed):
        if sharded:  # rows split across the ranks (strong scaling of one solve)
            eng = ShardedEngine(op, prob.partition, cfg, device=dev)
        else:
            eng = DeviceEngine(op, prob.partition, cfg, device=dev)
        eng.kernel_timer = timer
        timer.engine = eng
        timer.enabled = timed and not args.no_kernel_timer
        x, rep = eng.solve(b_dev)
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
    step_ms, iters, reps, dgram = [], 0, [], []
    n_rows = prob.n
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
        reps.append(rep)
        dgram.extend(kd for kd in eng.launch_k if kd[0] <= rep.iterations)
        n_rows = eng.n  # local rows on a shard
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
        it_t = torch.tensor([iters], device=dev, dtype=torch.float64)
        dist.all_reduce(it_t)
        # sharded: all ranks iterate the same solve; replicas: independent solves
        iters_all = int(it_t.item()) // world if sharded else int(it_t.item())
    else:
        iters_all = iters
    value = iters_all / (tot_ms / 1e3)

    # ---- roofline of the dominant kernel (algorithmic bytes / event-timed duration) ----
    m = prob.solver_kwargs["t"] * prob.solver_kwargs.get("s", 1)
    n = n_rows
    per_tag = {}
    for tag, k, d, mm, ms in timer.records:
        # Gram reads A Q_1..d and W; the update reads Q_1..d, W and writes W'
        bytes_ = 8.0 * (d + 1) * n * mm if tag == "hist_gram" else 8.0 * (d + 2) * n * mm
        flops = 2.0 * d * mm * mm * n
        acc = per_tag.setdefault(tag, [0.0, 0.0, 0.0, 0])
        acc[0] += bytes_
        acc[1] += flops
        acc[2] += ms
        acc[3] += 1
    dom = max(per_tag, key=lambda t: per_tag[t][2]) if per_tag else None
    hbm, peak_kind = peaks()
    achieved = per_tag[dom][0] / (per_tag[dom][2] / 1e3) / 1e9 if dom else None
    prof = ROOT / "profiles" / "r01_traffic.json"
    traffic, traffic_alg, traffic_d = None, None, None
    if prof.exists() and dom:
        tr = json.loads(prof.read_text())
        traffic, traffic_alg, traffic_d = tr.get(dom), tr.get(dom + "_alg"), tr.get(dom + "_d")
    model_bytes = sum(r.model_bytes for r in reps)
    model_time = model_bytes / (hbm * 1e9)
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
        "frac": (achieved / hbm) if achieved else None, "traffic": traffic, "kernel": dom,
        "traffic_alg_bytes": traffic_alg, "traffic_launch_d": traffic_d,
        "traffic_source": "profiles/r01_traffic.json (ncu --set full, one launch)",
        "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
        "per_kernel": {t: {"GBs": v[0] / (v[2] / 1e3) / 1e9, "TFLOPs": v[1] / (v[2] / 1e3) / 1e12,
                           "ms_total": round(v[2], 3), "launches": v[3]} for t, v in per_tag.items()},
        "timed_launches": f"CGS2 launches with d >= {timer.d_min} retained blocks, all timed steps",
        "step_model_gbs": model_bytes / (tot_ms / 1e3) / 1e9,
        "step_model_frac": model_time / (tot_ms / 1e3),
    }

    # ---- e2e through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        b_host = torch.from_numpy(np.ascontiguousarray(prob.b)).pin_memory()
        # The reference-facing call: the host CSR matrix a reference user holds (SparseSpdMatrix layout),
        # host b in, host x out -- the matrix upload, the operator set-up and the D2H are all timed.
        # A plain (n, row_ptr, col_idx, values) object like the reference's SparseSpdMatrix, so nothing is
        # cached on the device between calls: every call uploads the matrix.
        csr = prob.csr()
        A_host = types.SimpleNamespace(n=csr.n, row_ptr=csr.row_ptr, col_idx=csr.col_idx, values=csr.values)
        mat_bytes = 8 * (csr.n + 1) + 12 * csr.nnz
        # one untimed warm-up call of the public API path (first-call host costs)
        pk.enlarged_solve(A_host, b_host.numpy(), partition=prob.partition, cfg=cfg, device=dev)
        e2e_ms, e2e_it = [], 0
        for _ in range(max(1, args.steps)):
            flush.fill_(1.0)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            x, rep = pk.enlarged_solve(A_host, b_host.numpy(), partition=prob.partition, cfg=cfg, device=dev)
            e1.record()
            e1.synchronize()
            e2e_ms.append(e0.elapsed_time(e1))
            e2e_it += rep.iterations
        e2e_tot = sum(e2e_ms)
        if world > 1:
            t = torch.tensor([e2e_tot], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_tot = float(t.item())
            if not sharded:
                e2e_it *= world
        e2e = {"value": e2e_it / (e2e_tot / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * n + mat_bytes,
               "d2h_bytes_per_step": 8 * n + 8 * (reps[-1].iterations + 1),
               "call": "enlarged_solve(host CSR matrix, host numpy b) -> host x, report"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        it_cpu = args.cpu_iters or default_cpu_iters(args.config)
        its, dt = cpu_sample(make_config(args.config, args.edge, device_rhs=False), it_cpu)
        cpu = {"value": its / dt, "unit": UNIT, "cores": cores(), "kind": "port",
               "sample": f"first {it_cpu} of {reps[-1].iterations} iterations of {prob.name} "
                         f"(reference algorithm, numpy/OpenBLAS oracle port, {dt:.1f} s; early iterations "
                         f"are the cheapest, so this overstates CPU speed)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": prob.name, "form": args.form, "n": n, "t": prob.solver_kwargs["t"],
                       "s": prob.solver_kwargs.get("s", 1), "iterations_per_step": reps[-1].iterations,
                       "status": reps[-1].status,
                       "parallelism": (f"rows{world}" if sharded else "replicas") if world > 1 else "single",
                       "l2": "flushed (256 MB write) before every timed step",
                       "time_to_solution_ms": tot_ms / args.steps},
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
