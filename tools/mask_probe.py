"""Warm A/B of the ReLU bit mask on one box: forward with/without writing the mask, dX gated by
the mask vs by the bf16 tensor (CUDA events, back to back, min of 3 interleaved rounds)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

L = _capi.LIB
for rows, d in [(16384, 1600), (65792, 1280)]:
    x = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
    dz = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
    W = torch.randn(d, d, device="cuda").to(torch.bfloat16)
    bias = torch.randn(d, device="cuda")
    out = torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)
    mask = torch.zeros(rows * d // 32, device="cuda", dtype=torch.int32)
    st = torch.cuda.current_stream().cuda_stream
    M = mask.data_ptr()
    V = {
        "fwd": lambda: L.sp_debug_gemm_bf16_masked_async(rows, d, d, x.data_ptr(), d, 0, W.data_ptr(), d, 1, 0, out.data_ptr(), d, bias.data_ptr(), 1, None, 0, 1, 0, 0, st, None, None),
        "fwd+mask": lambda: L.sp_debug_gemm_bf16_masked_async(rows, d, d, x.data_ptr(), d, 0, W.data_ptr(), d, 1, 0, out.data_ptr(), d, bias.data_ptr(), 1, None, 0, 1, 0, 0, st, M, None),
        "dx(tensor gate)": lambda: L.sp_debug_gemm_bf16_masked_async(rows, d, d, dz.data_ptr(), d, 0, W.data_ptr(), d, 0, 2, out.data_ptr(), d, None, 1, x.data_ptr(), d, 1, 0, 0, st, None, None),
        "dx(mask gate)": lambda: L.sp_debug_gemm_bf16_masked_async(rows, d, d, dz.data_ptr(), d, 0, W.data_ptr(), d, 0, 2, out.data_ptr(), d, None, 1, x.data_ptr(), d, 1, 0, 0, st, None, M),
    }
    best = {}
    for _ in range(3):
        for k, fn in V.items():
            for _ in range(3):
                assert fn() == 0
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                fn()
            e1.record()
            e1.synchronize()
            best[k] = min(best.get(k, 1e9), e0.elapsed_time(e1) / 20 * 1e3)
    print(json.dumps({"rows": rows, "d": d, **{k: round(v, 1) for k, v in best.items()}}))
