"""Warm back-to-back timing (CUDA events, real clocks) of the step's GEMMs through the
product's auto dispatch, with the GEMM debug knobs epi_mode / narrow (sp_debug_set) taken from
the SP_EPI_MODE / SP_NARROW environment of this probe. Prints one JSON
line of microseconds per launch for each (rows, d, gemm). Used to pick the epilogue policy."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

LIB = _capi.LIB
out = {"env": {k: os.environ.get(k) for k in ("SP_EPI_MODE", "SP_NARROW")}}
LIB.sp_debug_set(None, b"epi_mode", int(os.environ.get("SP_EPI_MODE", "0")))
LIB.sp_debug_set(None, b"narrow", int(os.environ.get("SP_NARROW", "0")))
for rows, d in [(16384, 1600), (65792, 1280), (65536, 4096)]:
    x = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
    dz = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
    W = torch.randn(d, d, device="cuda").to(torch.bfloat16)
    bias = torch.randn(d, device="cuda")
    o = torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)
    splits = int(LIB.sp_debug_dw_splits(d, rows))
    parts = torch.empty(splits * d * d, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    fns = {
        "fwd": lambda: LIB.sp_debug_gemm_bf16_async(rows, d, d, x.data_ptr(), d, 0, W.data_ptr(), d, 1, 0,
                                                    o.data_ptr(), d, bias.data_ptr(), 1, None, 0, 1, 0, 0, st),
        "dx": lambda: LIB.sp_debug_gemm_bf16_async(rows, d, d, dz.data_ptr(), d, 0, W.data_ptr(), d, 0, 2,
                                                   o.data_ptr(), d, None, 1, x.data_ptr(), d, 1, 0, 0, st),
        "dw": lambda: LIB.sp_debug_gemm_bf16_async(d, d, rows, x.data_ptr(), d, 1, dz.data_ptr(), d, 1, 3,
                                                   parts.data_ptr(), d, None, 0, None, 0, splits, 0, 0, st),
    }
    reps = 20 if d < 4096 else 5
    for name, fn in fns.items():
        for _ in range(3):
            assert fn() == 0
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        out[f"{d}_{name}"] = round(e0.elapsed_time(e1) / reps * 1e3, 1)
print(json.dumps(out), flush=True)
