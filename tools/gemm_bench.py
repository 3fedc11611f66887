"""Times the tcgen05 GEMM variants (1-CTA M=128 tiles, 2-CTA cta_group::2 M=256 tiles, tile N)
on the three per-layer shapes of a square-block training step (forward, dX, dW-with-SGD) via
back-to-back launches between CUDA events, against torch.matmul (cuBLAS) as a yardstick.
Usage: python tools/gemm_bench.py [rows d]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

rows, d = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (16384, 1600)))
LIB = _capi.LIB
x = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
dz = (torch.randn(rows, d, device="cuda") * 1e-3).to(torch.bfloat16)
W = torch.randn(d, d, device="cuda").to(torch.bfloat16)
W32 = torch.randn(d, d, device="cuda")
bias = torch.randn(d, device="cuda")
out16 = torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)
SPLITS = int(LIB.sp_debug_dw_splits(d, rows))
parts = torch.empty(max(SPLITS, 1) * d * d, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def timeit(fn, reps=20):
    for _ in range(3):
        assert fn() == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


fl = 2.0 * rows * d * d
VARIANTS = [(1, 192), (1, 256), (2, 128), (2, 192), (2, 256), (0, 0)]
ROUNDS = int(os.environ.get("ROUNDS", "3"))


def shapes_for(cta, bn):
    return {
        "fwd": lambda: LIB.sp_debug_gemm_bf16_async(rows, d, d, x.data_ptr(), d, 0, W.data_ptr(), d, 1, 0,
                                                    out16.data_ptr(), d, bias.data_ptr(), 1, None, 0, 1,
                                                    bn, cta, st),
        "dx": lambda: LIB.sp_debug_gemm_bf16_async(rows, d, d, dz.data_ptr(), d, 0, W.data_ptr(), d, 0, 2,
                                                   out16.data_ptr(), d, None, 1, x.data_ptr(), d, 1, bn,
                                                   cta, st),
        "dw_sgd": lambda: LIB.sp_debug_gemm_bf16_async(d, d, rows, x.data_ptr(), d, 1, dz.data_ptr(), d, 1,
                                                       4, W32.data_ptr(), d, None, 0, None, 0, 1, bn, cta,
                                                       st),
        # dW as the executor runs it when one split underfills the SMs: split-K fp32 partials
        "dw_split": lambda: LIB.sp_debug_gemm_bf16_async(d, d, rows, x.data_ptr(), d, 1, dz.data_ptr(), d,
                                                         1, 3, parts.data_ptr(), d, None, 0, None, 0,
                                                         SPLITS, bn, cta, st),
    }


# Variants are interleaved round-robin over ROUNDS rounds (clock / power drift hits every
# variant alike); min and median per (variant, shape) are reported.
times = {}
for r in range(ROUNDS):
    for cta, bn in VARIANTS:
        for name, fn in shapes_for(cta, bn).items():
            if cta == 2 and bn == 192 and name != "dx":
                continue  # 2-CTA N=192 exists for K-major B only
            times.setdefault((cta, bn, name), []).append(timeit(fn))
for (cta, bn, name), ts in times.items():
    ts = sorted(ts)
    print(json.dumps({"cta": cta or "auto", "bn": bn or "auto", "gemm": name,
                      "ms_min": round(ts[0], 4), "ms_med": round(ts[len(ts) // 2], 4),
                      "tflops_best": round(fl / ts[0] / 1e9, 1)}), flush=True)
for name, fn in {"torch_fwd": lambda: torch.matmul(x, W),
                 "torch_dx": lambda: torch.matmul(dz, W.t()),
                 "torch_dw": lambda: torch.matmul(x.t(), dz)}.items():
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(json.dumps({"gemm": name, "ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1)}), flush=True)
