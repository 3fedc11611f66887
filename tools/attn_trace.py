"""Timeline of the tcgen05 dK/dV attention pass on CTA 0 (debug instantiation, sp_debug_set
"attn_trace"): per step, when the MMA issuer entered / issued the S and product MMAs and when each
softmax warpgroup entered the step, had S, and wrote P. Prints per-event gaps in SM clocks.
Usage: python tools/attn_trace.py [gpt2-xl|llama3-8b]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

LIB = _capi.LIB
SH = {"gpt2-xl": (16, 1024, 25, 25, 64, 1), "llama3-8b": (32, 2048, 32, 8, 128, 1), "vit-h14": (256, 257, 16, 16, 80, 0)}
B, S, H, Hkv, hd, causal = SH[sys.argv[1] if len(sys.argv) > 1 else "gpt2-xl"]
T, W = B * S, (H + 2 * Hkv) * hd
qkv = torch.randn(T, W, device="cuda").to(torch.bfloat16)
o = torch.empty(T, H * hd, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * S + 64, device="cuda")
dout = torch.randn(T, H * hd, device="cuda").to(torch.bfloat16)
dqkv = torch.empty_like(qkv)
delta = torch.empty(B * H * S + 64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
LIB.sp_debug_attention(0, T, S, H, Hkv, hd, causal, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), None, None, None, st)
LIB.sp_debug_attention(1, T, S, H, Hkv, hd, causal, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(),
                       delta.data_ptr(), dqkv.data_ptr(), st)
LIB.sp_debug_set(None, b"attn_trace", 1)
LIB.sp_debug_attention(1, T, S, H, Hkv, hd, causal, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(),
                       delta.data_ptr(), dqkv.data_ptr(), st)
torch.cuda.synchronize()
buf = np.zeros(4096, np.uint64)
n = LIB.sp_debug_attn_trace(buf.ctypes.data, 4096)
ev = [(int(v) >> 56, (int(v) >> 40) & 0xFFFF, int(v) & 0xFFFFFFFFFF) for v in buf[:n]]
t0 = min(e[2] for e in ev)
NAMES = {0: "S-enter", 1: "S-issue", 2: "D-enter", 3: "D-issue", 4: "wg0-enter", 5: "wg0-S", 6: "wg0-P",
         12: "wg1-enter", 13: "wg1-S", 14: "wg1-P"}
per = {}
for e, g, c in ev:
    per.setdefault(g, {})[NAMES.get(e, str(e))] = c - t0
steps = sorted(per)
rows = []
for g in steps[:60]:
    rows.append({"step": g, **per[g]})
for r in rows:
    print(json.dumps(r))
# summary: average durations over steps 4..end
def avg(a, b):
    xs = [per[g][b] - per[g][a] for g in steps if a in per[g] and b in per[g]]
    return round(float(np.mean(xs)), 1) if xs else None
wg = lambda g: "wg0" if g % 2 == 0 else "wg1"
sm = [per[g][wg(g) + "-P"] - per[g][wg(g) + "-S"] for g in steps if wg(g) + "-P" in per[g] and wg(g) + "-S" in per[g]]
wait = [per[g][wg(g) + "-S"] - per[g][wg(g) + "-enter"] for g in steps if wg(g) + "-S" in per[g] and wg(g) + "-enter" in per[g]]
dwait = [per[g]["D-issue"] - per[g]["D-enter"] for g in steps if "D-issue" in per[g] and "D-enter" in per[g]]
span = (max(e[2] for e in ev) - t0) / max(1, len(steps))
print(json.dumps({"events": n, "steps": len(steps), "clk_per_step": round(span, 1),
                  "softmax_compute_clk": round(float(np.mean(sm)), 1), "softmax_wait_S_clk": round(float(np.mean(wait)), 1),
                  "mma_wait_P_clk": round(float(np.mean(dwait)), 1),
                  "S_issue_wait_clk": avg("S-enter", "S-issue"), "S_issue_to_wgS": None}))
