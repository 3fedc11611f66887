"""Back-to-back named-shape train-step time through the block ABI (graphs on, device inputs), for
A/B of two library builds via SUPERPIPE_LIB: warm-up, then STEPS steps between CUDA events.
Usage: python tools/block_step_time.py [gpt2-xl] [steps] [seqs] [layers]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_08791_b200 as sp  # noqa: E402
from paper_2410_08791_b200 import _capi  # noqa: E402
from paper_2410_08791_b200 import blocks as B  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "gpt2-xl"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
spec, L = B.NAMED_SHAPES[name]
seqs = int(sys.argv[3]) if len(sys.argv) > 3 else 16
L = int(sys.argv[4]) if len(sys.argv) > 4 else L
model = B.build_block_model(spec, 7, L)
rows = seqs * spec.seq_len
x = torch.from_numpy(sp.make_input(7, 0, rows, spec.d)).cuda()
t = torch.from_numpy(sp.make_input(7, 1, rows, spec.d)).cuda()
ex = B.BlockExecutor(L, spec, sp.StrategyConfig(sp.SUPERPIPELINE, 4, 2), trace=0)
ex.register_model(model)
for _ in range(5):
    ex.train_step_ptr(x.data_ptr(), t.data_ptr(), rows, 0.01, device=True)
torch.cuda.synchronize()
res = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        ex.train_step_ptr(x.data_ptr(), t.data_ptr(), rows, 0.01, device=True)
    e1.record()
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / steps)
print(json.dumps({"lib": os.path.basename(_capi.LIB_PATH), "ms_per_step": [round(v, 2) for v in res]}))
