"""dX = (dz W^T) gated: warm back-to-back timing of the tcgen05 kernel variants against cuBLAS
at the C2 / C4 layer shapes (CUDA events)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_08791_b200 import _capi
LIB = _capi.LIB
for rows, d in [(16384, 1600), (65792, 1280), (65536, 4096)]:
    x = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
    dz = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
    W = torch.randn(d, d, device="cuda").to(torch.bfloat16)
    bias = torch.randn(d, device="cuda")
    out = torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)
    out32 = torch.empty(rows, d, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    fl = 2.0 * rows * d * d
    V = {
        "fwd_mnB_bias": lambda: LIB.sp_debug_gemm_bf16_async(rows, d, d, x.data_ptr(), d, 0, W.data_ptr(), d, 1, 0, out.data_ptr(), d, bias.data_ptr(), 1, None, 0, 1, 256, 2, st),
        "dx_kB_gate": lambda: LIB.sp_debug_gemm_bf16_async(rows, d, d, dz.data_ptr(), d, 0, W.data_ptr(), d, 0, 2, out.data_ptr(), d, None, 1, x.data_ptr(), d, 1, 256, 2, st),
        "dx_kB_nogate": lambda: LIB.sp_debug_gemm_bf16_async(rows, d, d, dz.data_ptr(), d, 0, W.data_ptr(), d, 0, 2, out.data_ptr(), d, None, 0, x.data_ptr(), d, 1, 256, 2, st),
        "kB_f32out": lambda: LIB.sp_debug_gemm_bf16_async(rows, d, d, dz.data_ptr(), d, 0, W.data_ptr(), d, 0, 3, out32.data_ptr(), d, None, 0, None, 0, 1, 256, 2, st),
        "mnB_f32out": lambda: LIB.sp_debug_gemm_bf16_async(rows, d, d, x.data_ptr(), d, 0, W.data_ptr(), d, 1, 3, out32.data_ptr(), d, None, 0, None, 0, 1, 256, 2, st),
    }
    res = {k: [] for k in V}
    for r in range(4):
        for k, fn in V.items():
            for _ in range(2): assert fn() == 0
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20): fn()
            e1.record(); e1.synchronize()
            res[k].append(e0.elapsed_time(e1) / 20)
    print(rows, d, json.dumps({k: round(fl / min(v) / 1e9) for k, v in res.items()}), flush=True)
