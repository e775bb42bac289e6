"""Can the HBM-bound stencil overlap the FP64-bound Gram?  Lean-scheme pass at config 5:
Y = A W (stencil) then C = [Q_1..Q_d]^T Y (Gram), sequential vs pipelined over row slabs on two streams.

    python tools/probe_overlap.py [edge] [slabs]
"""
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2305_19013_b200 import _lib  # noqa: E402
from paper_2305_19013_b200.problems import make_config  # noqa: E402

edge = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
S = int(sys.argv[2]) if len(sys.argv) > 2 else 8
prob = make_config(5, edge, device_rhs=False)
n, m, d = prob.n, 64, 3
op = prob.stencil("cuda")
dev = torch.device("cuda")
Qs = [torch.randn(n * m, dtype=torch.float64, device=dev) for _ in range(d)]
W = torch.randn(n * m, dtype=torch.float64, device=dev)
Y = torch.empty_like(W)
s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
plane = edge
planes_per = edge // S


def gram(rows0, rows, out, st):
    tab = torch.tensor([q.data_ptr() + 8 * rows0 * m for q in Qs], dtype=torch.int64, device=dev)
    chunks = _lib.query("ekcg_gram_chunks", rows, d, m, m)
    part = out[: chunks * d * m * m]
    _lib.call("ekcg_gram", tab.data_ptr(), m, d, m, Y.data_ptr() + 8 * rows0 * m, m, m, rows, part.data_ptr(), None,
              st.cuda_stream)
    return tab


def stencil(r0, r1, st):
    desc = type(op._desc)()
    ctypes.memmove(ctypes.byref(desc), ctypes.byref(op._desc), ctypes.sizeof(desc))
    desc.row_begin, desc.row_end = r0, r1
    assert _lib.query("ekcg_spmm_stencil", ctypes.byref(desc), W.data_ptr(), m, Y.data_ptr(), m, m, None,
                      st.cuda_stream) == 0


parts = [torch.empty(2048 * d * m * m, dtype=torch.float64, device=dev) for _ in range(S)]
whole = torch.empty(2048 * d * m * m, dtype=torch.float64, device=dev)
keep = []


def sequential():
    with torch.cuda.stream(s0):
        stencil(0, n, s0)
        keep.append(gram(0, n, whole, s0))


def pipelined():
    evs = []
    for s in range(S):
        r0, r1 = s * planes_per * plane, (s + 1) * planes_per * plane if s < S - 1 else n
        with torch.cuda.stream(s1):
            stencil(r0, r1, s1)
            ev = torch.cuda.Event()
            ev.record(s1)
        s0.wait_event(ev)
        with torch.cuda.stream(s0):
            keep.append(gram(r0, r1 - r0, parts[s], s0))
    s1.wait_stream(s0)


for name, f in (("sequential", sequential), ("pipelined", pipelined)) * 3:
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s0)
    s1.wait_stream(s0)
    f()
    s0.wait_stream(s1)
    e1.record(s0)
    e1.synchronize()
    keep.clear()
    print(f"edge {edge} slabs {S} {name}: {e0.elapsed_time(e1):.2f} ms", flush=True)
