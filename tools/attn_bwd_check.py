"""Attention backward check in a process of its own (a failing kernel poisons the context):
  python tools/attn_bwd_check.py KIND [B,S,H,Hkv,hd,causal]
runs the backward kind (sp_debug_set "attn_bwd") and prints rc and the max error of dQ, dK, dV
(relative to max |ref|) against autograd in fp32."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

LIB = _capi.LIB
kind = int(sys.argv[1])  # attn_bwd kind: 0 v2 tcgen05, 2 v1 tcgen05, 1 mma.sync
B, S, H, Hkv, hd, causal = (2, 1024, 4, 4, 64, 1) if len(sys.argv) < 3 else tuple(int(x) for x in sys.argv[2].split(","))
LIB.sp_debug_set(None, b"attn_bwd", kind)
T, W = B * S, (H + 2 * Hkv) * hd
qkv = torch.randn(T, W, device="cuda").to(torch.bfloat16)
o = torch.empty(T, H * hd, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * S, device="cuda")
st = torch.cuda.current_stream().cuda_stream
assert LIB.sp_debug_attention(0, T, S, H, Hkv, hd, causal, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), None, None, None, st) == 0
dout = torch.randn(T, H * hd, device="cuda").to(torch.bfloat16)
dqkv = torch.zeros(T, W, device="cuda", dtype=torch.bfloat16)
delta = torch.zeros(B * H * S, device="cuda")
rc = LIB.sp_debug_attention(1, T, S, H, Hkv, hd, causal, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(),
                            dout.data_ptr(), delta.data_ptr(), dqkv.data_ptr(), st)
torch.cuda.synchronize()
t = qkv.float().view(B, S, H + 2 * Hkv, hd).permute(0, 2, 1, 3)
q, k, v = (x.detach().requires_grad_(True) for x in (t[:, :H], t[:, H:H + Hkv], t[:, H + Hkv:]))
g = H // Hkv
kk, vv = k.repeat_interleave(g, 1), v.repeat_interleave(g, 1)
s = (q @ kk.transpose(-1, -2)) / math.sqrt(hd)
if causal:
    s = s.masked_fill(torch.triu(torch.ones(S, S, dtype=torch.bool, device="cuda"), 1), float("-inf"))
ref = torch.softmax(s, -1) @ vv
ref.backward(dout.float().view(B, S, H, hd).permute(0, 2, 1, 3))
got = dqkv.float().view(B, S, H + 2 * Hkv, hd).permute(0, 2, 1, 3)
out = {"kind": kind, "shape": (B, S, H, Hkv, hd, causal), "rc": rc}
for name, gg, rr in (("dq", got[:, :H], q.grad), ("dk", got[:, H:H + Hkv], k.grad), ("dv", got[:, H + Hkv:], v.grad)):
    out[name] = float((gg - rr).abs().max() / rr.abs().max())
print(out, flush=True)
