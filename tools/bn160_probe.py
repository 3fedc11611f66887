"""Narrower CTA-pair tiles against wave quantization: dX at 16384 x 1600 (and 65792 x 1280) with
N = 256 / 192 / 160 tiles, warm back-to-back CUDA-event timing (rejected)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_08791_b200 import _capi
L = _capi.LIB
for rows, d in [(16384, 1600), (65792, 1280)]:
    dz = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
    W = torch.randn(d, d, device="cuda").to(torch.bfloat16)
    x = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
    out = torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)
    mask = torch.zeros(rows * d // 32, device="cuda", dtype=torch.int32)
    st = torch.cuda.current_stream().cuda_stream
    res = {}
    for _ in range(3):
        for cta, bn in [(2, 256), (2, 192), (2, 160), (0, 0)]:
            fn = lambda: L.sp_debug_gemm_bf16_masked_async(rows, d, d, dz.data_ptr(), d, 0, W.data_ptr(), d, 0, 2, out.data_ptr(), d, None, 1, x.data_ptr(), d, 1, bn, cta, st, None, mask.data_ptr())
            if fn() != 0:
                continue
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20): fn()
            e1.record(); e1.synchronize()
            k = f"{cta}x{bn}"
            res[k] = min(res.get(k, 1e9), e0.elapsed_time(e1) / 20 * 1e3)
    print(rows, d, json.dumps({k: round(v, 1) for k, v in res.items()}))
