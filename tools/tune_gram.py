"""Time ekcg_gram / ekcg_block_update at config-2 sizes for the tuning variants."""
import sys, json
import torch
sys.path.insert(0, '.')
from paper_2305_19013_b200 import _lib

n, m = 262144, 16
dev = 'cuda'
res = {}
for d in (8, 32, 110):
    Xs = [torch.randn(n, m, dtype=torch.float64, device=dev) for _ in range(d)]
    Y = torch.randn(n, m, dtype=torch.float64, device=dev)
    tab = torch.tensor([x.data_ptr() for x in Xs], dtype=torch.int64, device=dev)
    part = torch.empty(4 * 4096 * 4 * m * m, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    for v in range(7):
        for target in (592, 1184, 2368):
            _lib.call('ekcg_tune', 1, v); _lib.call('ekcg_tune', 2, target)
            ch = _lib.query('ekcg_gram_chunks', n, d, m, m)
            for _ in range(3):
                _lib.call('ekcg_gram', tab.data_ptr(), m, d, m, Y.data_ptr(), m, m, n, part.data_ptr(), None, st)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                _lib.call('ekcg_gram', tab.data_ptr(), m, d, m, Y.data_ptr(), m, m, n, part.data_ptr(), None, st)
            e1.record(); e1.synchronize()
            ms = e0.elapsed_time(e1) / 10
            gbs = (d + 1) * n * m * 8 / ms / 1e6
            res[f'd{d}_v{v}_t{target}'] = (round(ms * 1e3, 1), round(gbs))
            print(f'd={d} v={v} target={target} chunks={ch}: {ms*1e3:.1f} us {gbs:.0f} GB/s', flush=True)
    del Xs
_lib.call('ekcg_tune', 1, -1); _lib.call('ekcg_tune', 2, 0)
json.dump(res, open('gpurun_out/tune_gram.json', 'w'), indent=1)
