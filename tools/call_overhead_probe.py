"""Host-side cost of one small inference call (C1, 12 x d=768, 4 items x 1 row, SP(2,1), item
batching): wall time per call vs the device makespan, and the time spent enqueuing.
Usage: python tools/call_overhead_probe.py"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_08791_b200 as sp  # noqa: E402
from paper_2410_08791_b200 import _capi  # noqa: E402

n, d, items, rows = 12, 768, 4, 1
ex = sp.Executor(n, d, sp.StrategyConfig(sp.SUPERPIPELINE, 2, 1), numerics=sp.BF16, trace=0)
W = np.empty((d, d), np.float32)
b = np.empty((d,), np.float32)
for i in range(n):
    _capi.LIB.sp_build_layer(7, i, d, 0, 0, W.ctypes.data, b.ctypes.data)
    ex.register_layer(i, W, b)
ex.set_item_batching(True)
x = torch.from_numpy(np.stack([sp.make_input(7, i, rows, d) for i in range(items)])).cuda()
y = torch.empty_like(x)
for _ in range(20):
    ex.forward_ptr(x.data_ptr(), rows, items, y.data_ptr(), device=True)
torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
mk, enq = [], []
for _ in range(N):
    ex.forward_ptr(x.data_ptr(), rows, items, y.data_ptr(), device=True)
    st = ex.stats()
    mk.append(st["makespan_ms"])
    enq.append(st["host_enqueue_ms"])
wall = (time.perf_counter() - t0) / N * 1e3
print(json.dumps({"wall_ms_per_call": wall, "device_makespan_ms": float(np.median(mk)),
                  "host_enqueue_ms": float(np.median(enq)),
                  "host_gap_ms": wall - float(np.median(mk))}))
