"""Interleaved A/B of process-wide kernel knobs (sp_debug_set: "narrow", "epi_mode", "attn_fwd",
"attn_bwd") on the named-shape training step: one executor, graphs off (a knob does not change
the call signature, so a captured graph would replay the old choice), ROUNDS x (arm A, arm B),
STEPS steps each between CUDA events; prints the per-arm median.
Usage: python tools/block_ab.py KEY VALUE_A VALUE_B [--model gpt2-xl --layers 48 --seqs 16]"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_08791_b200 as sp  # noqa: E402
from paper_2410_08791_b200 import _capi  # noqa: E402
from paper_2410_08791_b200 import blocks as B  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("key")
p.add_argument("a", type=int)
p.add_argument("b", type=int)
p.add_argument("--model", default="gpt2-xl")
p.add_argument("--layers", type=int, default=0)
p.add_argument("--seqs", type=int, default=16)
p.add_argument("--rounds", type=int, default=4)
p.add_argument("--steps", type=int, default=4)
a = p.parse_args()
spec, L = B.NAMED_SHAPES[a.model]
L = a.layers or L
model = B.build_block_model(spec, 7, L)
rows = a.seqs * spec.seq_len
x = torch.from_numpy(sp.make_input(7, 0, rows, spec.d)).cuda()
t = torch.from_numpy(sp.make_input(7, 1, rows, spec.d)).cuda()
ex = B.BlockExecutor(L, spec, sp.StrategyConfig(sp.SUPERPIPELINE, 4, 2), trace=0)
ex.register_model(model)
ex.debug_set("graphs", 0)
LIB = _capi.LIB


def run(v):
    assert LIB.sp_debug_set(None, a.key.encode(), v) == 0
    ex.train_step_ptr(x.data_ptr(), t.data_ptr(), rows, 0.01, device=True)  # warm with this setting
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        ex.train_step_ptr(x.data_ptr(), t.data_ptr(), rows, 0.01, device=True)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.steps


res = {a.a: [], a.b: []}
for _ in range(a.rounds):
    for v in (a.a, a.b):
        res[v].append(run(v))
print(json.dumps({"key": a.key, "model": a.model, "ms_per_step": {str(k): round(statistics.median(v), 2) for k, v in res.items()},
                  "all": {str(k): [round(x, 2) for x in v] for k, v in res.items()}}))
