import sys, json, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2305_19013_b200 as pk
from test_precond import _factor, CASES
meta = json.load(open('/root/repo/tests/golden/precond.json')); arrays = dict(np.load('/root/repo/tests/golden/precond.npz'))
for name in CASES:
    ref = meta[name]; A, F = _factor(meta, arrays, name); kw = dict(ref['cfg'])
    p = pk.contiguous_partition(A.n, kw['t'])
    x, rep = pk.enlarged_solve(A, arrays[f"{name}__b"], x0=arrays.get(f"{name}__x0"), partition=p, cfg=pk.SolverConfig(preconditioner=F, **kw))
    h, g = rep.residual_history, arrays[f"{name}__history"]
    n = min(len(h), len(g), 21)
    d = np.abs(h[:n] / h[0] - g[:n] / g[0]) / (g[:n] / g[0])
    print(name, rep.iterations, ref['iterations'], ' '.join(f"{v:.0e}" for v in d[:12]))
