"""Device time of the one-kernel cluster solve (ekcg_cluster_solve) against the whole
enlarged_solve call and the launch-per-phase engine, on config-1-class problems.

    python tools/cluster_time.py [--edges 100,64,200] [--repeats 5]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2305_19013_b200 as pk  # noqa: E402
from paper_2305_19013_b200 import _lib  # noqa: E402
from paper_2305_19013_b200.engine import DeviceEngine  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402


PHASES = ['candidate', 'cgs2_gram', 'cgs2_sum', 'cgs2_update', 'graw_gram', 'graw_sum', 'prechol', 'w0_tri+sync',
          'apply_w0', 'g_gram', 'g_sum', 'cholinv', 'wk_tri', 'alpha_gram', 'alpha_sum', 'apply_wk', 'xr', 'rho_sum',
          'check']


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--edges", default="100")
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--over", default="{}")
    ap.add_argument("--phases", action="store_true", help="per-phase SM cycles of CTA 0")
    args = ap.parse_args()
    over = json.loads(args.over)
    real_call = _lib.call
    kernel_ms = []

    def timed_call(name, *a):
        if name != "ekcg_cluster_solve":
            return real_call(name, *a)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = real_call(name, *a)
        e1.record()
        e1.synchronize()
        kernel_ms.append(e0.elapsed_time(e1))
        return rc

    import paper_2305_19013_b200.engine as eng_mod
    for edge in [int(e) for e in args.edges.split(",")]:
        prob = make_config(args.config, edge)
        cfg = pk.SolverConfig(**dict(prob.solver_kwargs, **over))
        op = prob.stencil()
        b = torch.as_tensor(prob.b, device="cuda")
        out = {"config": prob.name, "n": prob.n, "t": cfg.t}
        for use in (True, False):
            best = None
            for _ in range(args.repeats):
                eng = DeviceEngine(op, prob.partition, cfg)
                eng.use_cluster = use
                if use and args.phases:
                    eng.cluster_ticks = torch.zeros(20, dtype=torch.int64, device='cuda')
                kernel_ms.clear()
                eng_mod._lib.call = timed_call
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                x, rep = eng.solve(b)
                e1.record()
                e1.synchronize()
                eng_mod._lib.call = real_call
                ms = e0.elapsed_time(e1)
                km = kernel_ms[0] if kernel_ms else None
                if best is None or ms < best[0]:
                    best = (ms, km, rep.iterations, rep.solve_seconds * 1e3)
                    if use and args.phases:
                        ticks = eng.cluster_ticks.cpu().numpy()
                        out['phase_cycles_per_iteration'] = {PHASES[i]: round(float(ticks[i]) / rep.iterations, 1)
                                                             for i in range(len(PHASES))}
            key = "cluster" if use else "launches"
            out[key] = {"call_ms": round(best[0], 3), "solve_ms": round(best[3], 3), "iterations": best[2],
                        "kernel_ms": None if best[1] is None else round(best[1], 3),
                        "us_per_iteration": round(1e3 * (best[1] if best[1] else best[3]) / best[2], 2)}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
