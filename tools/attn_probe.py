"""Attention-core timing at the named shapes: this repo's kernels (sp_debug_attention) against
torch's scaled_dot_product_attention (library kernels, context only) on the same bf16 inputs.
Prints one JSON line per shape: us per launch and TFLOP/s (causal FLOPs counted as half)."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

LIB = _capi.LIB
# SP_ATTN_FWD=0|1|3: the forward kernel choice (sp_debug_set "attn_fwd"; 0 = v2 tcgen05, 3 = v1, 1 = mma.sync)
LIB.sp_debug_set(None, b"attn_fwd", int(os.environ.get("SP_ATTN_FWD", "0")))
LIB.sp_debug_set(None, b"attn_bwd", int(os.environ.get("SP_ATTN_BWD", "0")))
# SP_ATTN_CHUNK=N: (sequence, head) pairs per chunk of the causal work order (0 = by shape)
LIB.sp_debug_set(None, b"attn_chunk", int(os.environ.get("SP_ATTN_CHUNK", "0")))


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


SHAPES = [("gpt2-xl", 16, 1024, 25, 25, 64, 1), ("vit-h14", 256, 257, 16, 16, 80, 0),
          ("llama3-8b", 32, 2048, 32, 8, 128, 1)]
for name, B, S, H, Hkv, hd, causal in SHAPES:
    if len(sys.argv) > 1 and name not in sys.argv[1:]:
        continue
    T, W = B * S, (H + 2 * Hkv) * hd
    qkv = torch.randn(T, W, device="cuda").to(torch.bfloat16)
    o = torch.empty(T, H * hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    dout = torch.randn(T, H * hd, device="cuda").to(torch.bfloat16)
    dqkv = torch.empty_like(qkv)
    delta = torch.empty(B * H * S, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    fwd = lambda: LIB.sp_debug_attention(0, T, S, H, Hkv, hd, causal, qkv.data_ptr(), o.data_ptr(),  # noqa: E731
                                         lse.data_ptr(), None, None, None, st)
    bwd = lambda: LIB.sp_debug_attention(1, T, S, H, Hkv, hd, causal, qkv.data_ptr(), o.data_ptr(),  # noqa: E731
                                         lse.data_ptr(), dout.data_ptr(), delta.data_ptr(), dqkv.data_ptr(), st)
    keys = (S + 1) / 2 if causal else S
    fl = 4.0 * T * keys * hd * H
    out = {"shape": name, "ours_fwd_us": timeit(fwd), "ours_bwd_us": timeit(bwd)}
    out["ours_fwd_tflops"] = fl / out["ours_fwd_us"] / 1e6
    out["ours_bwd_tflops"] = 2.5 * fl / out["ours_bwd_us"] / 1e6  # dQ, dK, dV, dP, S recompute
    q = qkv.view(B, S, H + 2 * Hkv, hd)[:, :, :H].permute(0, 2, 1, 3).contiguous().requires_grad_(True)
    k = qkv.view(B, S, H + 2 * Hkv, hd)[:, :, H:H + Hkv].permute(0, 2, 1, 3).contiguous().requires_grad_(True)
    v = qkv.view(B, S, H + 2 * Hkv, hd)[:, :, H + Hkv:].permute(0, 2, 1, 3).contiguous().requires_grad_(True)
    try:
        f = lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=bool(causal),  # noqa: E731
                                                                     enable_gqa=Hkv != H)
        out["sdpa_fwd_us"] = timeit(f)
        y = f()
        g = torch.randn_like(y)
        out["sdpa_bwd_us"] = timeit(lambda: torch.autograd.grad(y, (q, k, v), g, retain_graph=True))
        out["sdpa_fwd_tflops"] = fl / out["sdpa_fwd_us"] / 1e6
        out["sdpa_bwd_tflops"] = 2.5 * fl / out["sdpa_bwd_us"] / 1e6
    except Exception as e:  # noqa: BLE001
        out["sdpa_error"] = str(e)[:200]
    print(json.dumps(out), flush=True)
