"""Times the tcgen05 GEMM (sp_debug_gemm_bf16) on the three per-layer shapes of a square
block training step (forward, dX, dW) for each tile width, against torch.matmul (cuBLAS)
as a yardstick. CUDA events on the default stream; L2 flushed between launches.
Usage: python tools/gemm_bench.py [rows d]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

rows, d = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (16384, 1600)))
LIB = _capi.LIB
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
x = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
dz = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
W = torch.randn(d, d, device="cuda").to(torch.bfloat16)
bias = torch.randn(d, device="cuda")
out16 = torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)
out32 = torch.empty(16 * d * d, device="cuda", dtype=torch.float32)


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps


res = []
for bn in (128, 192, 256):
    shapes = {
        "fwd": lambda: LIB.sp_debug_gemm_bf16(rows, d, d, x.data_ptr(), d, 0, W.data_ptr(), d, 1, 0,
                                              out16.data_ptr(), d, bias.data_ptr(), 1, None, 0, 1, bn),
        "dx": lambda: LIB.sp_debug_gemm_bf16(rows, d, d, dz.data_ptr(), d, 0, W.data_ptr(), d, 0, 2,
                                             out16.data_ptr(), d, None, 1, x.data_ptr(), d, 1, bn),
    }
    for s in (1, 2, 4, 6, 8):
        shapes[f"dw_s{s}"] = (lambda s=s: LIB.sp_debug_gemm_bf16(
            d, d, rows, x.data_ptr(), d, 1, dz.data_ptr(), d, 1, 3, out32.data_ptr(), d, None, 0,
            None, 0, s, bn))
    for name, fn in shapes.items():
        ms = timeit(fn)
        fl = 2.0 * rows * d * d
        res.append({"bn": bn, "gemm": name, "ms": ms, "tflops": fl / ms / 1e9})
        print(json.dumps(res[-1]), flush=True)
for name, fn in {"torch_fwd": lambda: torch.matmul(x, W),
                 "torch_dx": lambda: torch.matmul(dz, W.t()),
                 "torch_dw": lambda: torch.matmul(x.t(), dz)}.items():
    ms = timeit(fn)
    print(json.dumps({"gemm": name, "ms": ms, "tflops": 2.0 * rows * d * d / ms / 1e9}), flush=True)
