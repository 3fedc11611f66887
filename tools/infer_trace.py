"""Per-op measured timeline (trace=1) of one Superpipeline inference call, to see copy/compute
overlap and gaps. Usage: python tools/infer_trace.py n d items rows k kp"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_08791_b200 as sp  # noqa: E402
from paper_2410_08791_b200 import _capi  # noqa: E402

n, d, items, rows, k, kp = (int(v) for v in sys.argv[1:7])
ex = sp.Executor(n, d, sp.StrategyConfig(sp.SUPERPIPELINE, k, kp), numerics=sp.BF16, trace=1)
W = np.empty((d, d), np.float32)
b = np.empty((d,), np.float32)
for i in range(n):
    _capi.LIB.sp_build_layer(7, i, d, 0, 0, W.ctypes.data, b.ctypes.data)
    ex.register_layer(i, W, b)
x = torch.from_numpy(np.stack([sp.make_input(7, i, rows, d) for i in range(items)])).cuda()
y = torch.empty_like(x)
for _ in range(4):
    ex.forward_ptr(x.data_ptr(), rows, items, y.data_ptr(), device=True)
st = ex.stats()
print({k: st[k] for k in ("makespan_ms", "compute_ms", "stall_ms", "h2d_bytes", "graph_replays",
                          "host_enqueue_ms")})
for e in ex.trace()[:40]:
    print(f"{e['kind']:8s} L{e['layer']:3d} first={e['first_layer']:3d} n={e['n_layers_moved']} "
          f"[{e['t_start'] * 1e3:9.1f}, {e['t_end'] * 1e3:9.1f}] us  dur={(e['t_end'] - e['t_start']) * 1e3:7.1f}")
