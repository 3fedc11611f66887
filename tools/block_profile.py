"""One named-shape training step for ncu's launch list: warm-up steps outside the profiled
range, then exactly one step between cudaProfilerStart / Stop. Run as
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file launches.csv python tools/block_profile.py [--model gpt2-xl --layers 48 --seqs 16]
(graphs are disabled so every kernel is a plain launch in stream order)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_08791_b200 as sp  # noqa: E402
from paper_2410_08791_b200 import _capi  # noqa: E402
from paper_2410_08791_b200 import blocks as B  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--model", default="gpt2-xl")
p.add_argument("--layers", type=int, default=0)
p.add_argument("--seqs", type=int, default=16)
p.add_argument("--k", type=int, default=4)
p.add_argument("--kp", type=int, default=2)
p.add_argument("--infer", action="store_true")
p.add_argument("--ckpt", action="store_true")
p.add_argument("--graphs", type=int, default=0)
p.add_argument("--set", action="append", default=[], help="KEY=VALUE process-wide kernel knob (sp_debug_set)")
a = p.parse_args()
spec, L = B.NAMED_SHAPES[a.model]
L = a.layers or L
model = B.build_block_model(spec, 7, L)
rows = a.seqs * spec.seq_len
x = torch.from_numpy(sp.make_input(7, 0, rows, spec.d)).cuda()
t = torch.from_numpy(sp.make_input(7, 1, rows, spec.d)).cuda()
y = torch.empty_like(x)
ex = B.BlockExecutor(L, spec, sp.StrategyConfig(sp.SUPERPIPELINE, a.k, a.kp), checkpointing=a.ckpt, trace=0)
ex.register_model(model)
ex.debug_set("graphs", a.graphs)
for kv in a.set:
    k, v = kv.split("=")
    assert _capi.LIB.sp_debug_set(None, k.encode(), int(v)) == 0, kv


def step():
    if a.infer:
        ex.forward_ptr(x.data_ptr(), rows, 1, y.data_ptr(), device=True)
    else:
        ex.train_step_ptr(x.data_ptr(), t.data_ptr(), rows, 0.01, device=True)


for _ in range(3):
    step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("stats", {k: v for k, v in ex.stats().items() if k in ("makespan_ms", "kernels_launched", "gemm_launches")})
