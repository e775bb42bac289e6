"""A/B timing of full config solves: fused vs unfused, with/without the bench kernel timer."""
import sys, time, json
import torch
sys.path.insert(0, '.')
import paper_2305_19013_b200 as pk
from paper_2305_19013_b200.engine import DeviceEngine
from paper_2305_19013_b200.problems import make_config
import bench

cfg_idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prob = make_config(cfg_idx)
cfg = pk.SolverConfig(**prob.solver_kwargs)
op = prob.stencil()
b = torch.as_tensor(prob.b, device='cuda')
timer = bench.KernelTimer(torch, ["hist_gram", "hist_update"])
variants = [("none", set()), ("cholinv+vec", {"cholinv", "vec"}), ("vec+xr", {"vec", "xr"}),
            ("vec", {"vec"}), ("default", None)]
for name, fuse in variants:
    for timed in (False,):
        ms = []
        for rep in range(4):
            eng = DeviceEngine(op, prob.partition, cfg)
            if fuse is not None:
                eng.fuse = fuse
            eng.kernel_timer = timer
            timer.engine = eng
            timer.enabled = timed
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            x, r = eng.solve(b)
            e1.record(); e1.synchronize()
            timer.harvest(r.iterations)
            ms.append(e0.elapsed_time(e1))
        print(f"fuse={name} timed={timed}: iters={r.iterations} ms={[round(v,1) for v in ms]} timer_records={len(timer.records)}", flush=True)
        timer.records = []
