"""Back-to-back train-step time through the core ABI only (works with any libsuperpipe build,
for A/B via SUPERPIPE_LIB): warmup, then K steps between CUDA events on the current stream.
Usage: python tools/step_time.py [layers d rows k kp steps]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_08791_b200 as sp  # noqa: E402
from paper_2410_08791_b200 import _capi  # noqa: E402

L, d, rows, k, kp, steps = (int(v) for v in (sys.argv[1:7] if len(sys.argv) > 6 else (48, 1600, 16384, 4, 2, 10)))
strat = sp.StrategyConfig(sp.STANDARD) if k == 0 else sp.StrategyConfig(sp.SUPERPIPELINE, k, kp)  # k=0: Standard
ex = sp.Executor(L, d, strat, numerics=sp.BF16, trace=0)
W = np.empty((d, d), np.float32)
b = np.empty((d,), np.float32)
for i in range(L):
    _capi.LIB.sp_build_layer(7, i, d, 0, 0, W.ctypes.data, b.ctypes.data)
    ex.register_layer(i, W, b)
if os.environ.get("OPT") == "adamw":  # the AdamW variant of the step
    ex.set_optimizer(sp.OPT_ADAMW, 0.9, 0.999, 1e-8, 0.01)
x = torch.from_numpy(sp.make_input(7, 0, rows, d)).cuda()
t = torch.from_numpy(sp.make_input(7, 1, rows, d)).cuda()
for _ in range(3):
    ex.train_step_ptr(x.data_ptr(), t.data_ptr(), rows, 0.01, device=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(steps):
    loss = ex.train_step_ptr(x.data_ptr(), t.data_ptr(), rows, 0.01, device=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
st = ex.stats()
print(json.dumps({"lib": os.path.basename(_capi.LIB_PATH), "ms_per_step": round(ms, 3),
                  "samples_per_s": round(rows / ms * 1e3), "device_makespan_ms": round(st["makespan_ms"], 3),
                  "host_enqueue_ms": round(st["host_enqueue_ms"], 3), "loss": loss}))
