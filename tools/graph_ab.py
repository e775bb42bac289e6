import sys, time, torch
sys.path.insert(0, '.')
import paper_2305_19013_b200 as pk
from paper_2305_19013_b200.engine import DeviceEngine
from paper_2305_19013_b200.problems import make_config
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prob = make_config(idx)
cfg = pk.SolverConfig(**prob.solver_kwargs)
op = prob.stencil()
b = torch.as_tensor(prob.b, device='cuda')
for graphs in (False, True, False, True):
    for rep in range(3):
        eng = DeviceEngine(op, prob.partition, cfg)
        eng.use_graphs = graphs
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x, r = eng.solve(b)
        e1.record(); e1.synchronize()
        print(f"graphs={graphs} iters={r.iterations} dev_ms={e0.elapsed_time(e1):.1f} wall_ms={(time.perf_counter()-t0)*1e3:.1f} captured={len(eng._graphs or {})}", flush=True)
