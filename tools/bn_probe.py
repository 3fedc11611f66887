"""2-CTA tile width at the GPT-2 XL block's N = d GEMMs: the dX-style ones (K-major B) at N = 256
(ragged last tile) against N = 160 / 192 (whole tiles at d = 1600), and the forward's MN-major
residual / QKV projections (MN-major B) at N = 256 only: a 192-wide variant with 64B-swizzled B
halves was measured here and dropped (bitwise equal, 6-12% slower: 283 -> 312 us at FC2);
outputs checked bitwise equal across widths. Back-to-back launches between CUDA events, interleaved
rounds, median; one JSON line per shape / epilogue.
Usage: python tools/bn_probe.py"""
import ctypes as C
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

LIB = _capi.LIB
BIAS_BF16, GATE_BF16, F32, RESID_F32 = 0, 2, 3, 6
st = torch.cuda.current_stream().cuda_stream


def timeit(args, reps=20):
    for _ in range(3):
        assert LIB.sp_debug_gemm_ex(C.byref(args)) == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        LIB.sp_debug_gemm_ex(C.byref(args))
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for (M, N, K) in ((16384, 1600, 1600), (16384, 1600, 6400), (16384, 1600, 4800)):
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)  # K-major B
    for epi, out in ((GATE_BF16, torch.empty(M, N, device="cuda", dtype=torch.bfloat16)),
                     (F32, torch.empty(M, N, device="cuda"))):
        ref = None
        res = {}
        for bn in (256, 192, 160):
            args = _capi.GemmArgs(M, N, K, a.data_ptr(), K, 0, w.data_ptr(), K, 0, epi, out.data_ptr(), N,
                                  None, 0, None, 0, 1, bn, 2, None, 0, 0, st)
            assert LIB.sp_debug_gemm_ex(C.byref(args)) == 0
            torch.cuda.synchronize()
            if ref is None:
                ref = out.float().clone()
            else:
                assert torch.equal(out.float(), ref), f"bn={bn} differs"
            res[bn] = args
        t = {bn: [] for bn in res}
        for _ in range(4):
            for bn, args in res.items():
                t[bn].append(timeit(args))
        us = {bn: round(statistics.median(v), 1) for bn, v in t.items()}
        print(json.dumps({"M": M, "N": N, "K": K, "epi": epi, "us": us,
                          "tflops": {bn: round(2.0 * M * N * K / u / 1e6) for bn, u in us.items()}}), flush=True)


bf = torch.bfloat16
for (M, N, K, epi) in ((16384, 1600, 6400, RESID_F32), (16384, 1600, 1600, RESID_F32), (16384, 4800, 1600, BIAS_BF16)):
    a = torch.randn(M, K, device="cuda").to(bf)
    w = (torch.randn(K, N, device="cuda") * 0.02).to(bf)  # [K][N]: MN-major B
    bias = torch.randn(N, device="cuda")
    resid = torch.randn(M, N, device="cuda") if epi == RESID_F32 else None
    out = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi == RESID_F32 else bf)
    ref, res = None, {}
    for bn in (256,):
        args = _capi.GemmArgs(M, N, K, a.data_ptr(), K, 0, w.data_ptr(), N, 1, epi, out.data_ptr(), N,
                              bias.data_ptr(), 0, resid.data_ptr() if resid is not None else None, N if resid is not None else 0,
                              1, bn, 2, None, 0, 0, st)
        assert LIB.sp_debug_gemm_ex(C.byref(args)) == 0
        torch.cuda.synchronize()
        if ref is None:
            ref = out.float().clone()
            exp = a.float() @ w.float() + bias + (resid if resid is not None else 0)
            print(json.dumps({"check_vs_fp32": float((ref - exp).norm() / exp.norm())}))
        else:
            assert torch.equal(out.float(), ref), f"bn={bn} differs"
        res[bn] = args
    t = {bn: [] for bn in res}
    for _ in range(4):
        for bn, args in res.items():
            t[bn].append(timeit(args))
    us = {bn: round(statistics.median(v), 1) for bn, v in t.items()}
    print(json.dumps({"M": M, "N": N, "K": K, "epi": epi, "b": "mn", "us": us,
                      "tflops": {bn: round(2.0 * M * N * K / u / 1e6) for bn, u in us.items()}}), flush=True)
