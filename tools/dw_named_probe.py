"""dW split-K sweep at the GPT-2 XL block's four weight shapes (16 x 1024 tokens): the CTA-pair
tcgen05 GEMM with fp32 partials, 1..6 splits, against the split count choose_dw picks
(sp_debug_set-free: explicit splits through sp_debug_gemm_ex). Back-to-back launches between
CUDA events, interleaved rounds; prints one JSON line per shape.
Usage: python tools/dw_named_probe.py"""
import ctypes as C
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

LIB = _capi.LIB
T = 16384
st = torch.cuda.current_stream().cuda_stream
SHAPES = {"Wqkv": (1600, 4800), "Wo": (1600, 1600), "W1": (1600, 6400), "W2": (6400, 1600)}


def gemm_args(M, N, x, dy, parts, splits):
    return _capi.GemmArgs(M, N, T, x.data_ptr(), M, 1, dy.data_ptr(), N, 1, 3, parts.data_ptr(), N, None, 0, None, 0,
                          splits, 256, 2, None, 0, 0, st)


def timeit(args, reps=10):
    for _ in range(2):
        assert LIB.sp_debug_gemm_ex(C.byref(args)) == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        LIB.sp_debug_gemm_ex(C.byref(args))
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for name, (M, N) in SHAPES.items():
    x = torch.randn(T, M, device="cuda").to(torch.bfloat16)
    dy = (torch.randn(T, N, device="cuda") * 1e-2).to(torch.bfloat16)
    parts = torch.empty(6 * M * N, device="cuda")
    res = {s: [] for s in range(1, 7)}
    for _ in range(3):
        for s in range(1, 7):
            res[s].append(timeit(gemm_args(M, N, x, dy, parts, s)))
    us = {s: round(statistics.median(v), 1) for s, v in res.items()}
    print(json.dumps({"shape": name, "M": M, "N": N, "K": T, "us_by_splits": us,
                      "tflops_best": round(2.0 * M * N * T / min(us.values()) / 1e6, 1)}), flush=True)
