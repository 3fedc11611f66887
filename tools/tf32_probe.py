"""tf32 layer GEMMs (tcgen05 kind::tf32) at a layer shape: forward (bias+ReLU+mask, fp32 out),
dX (mask-gated, fp32 out), dW (split-K fp32 partials, the executor's choose_dw), each timed over
back-to-back launches with CUDA events, against cuBLAS tf32 (torch.matmul with tf32 allowed) of
the same product. Usage: python tools/tf32_probe.py [rows d]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

LIB = _capi.LIB
rows, d = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (16384, 1600)))
x = torch.randn(rows, d, device="cuda")
W = torch.randn(d, d, device="cuda") * 0.02
dz = torch.randn(rows, d, device="cuda")
bias = torch.randn(d, device="cuda")
y = torch.empty(rows, d, device="cuda")
mask = torch.empty(d // 32, rows, dtype=torch.int32, device="cuda")
cta = _capi.C.c_int32()
bn = _capi.C.c_int32()
splits = LIB.sp_debug_dw_choice(d, rows, 0, _capi.C.byref(cta), _capi.C.byref(bn))
parts = torch.empty(splits * d, d, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def fwd():
    return LIB.sp_debug_gemm_tf32_async(rows, d, d, x.data_ptr(), d, 0, W.data_ptr(), d, 1, 1, y.data_ptr(), d,
                                        bias.data_ptr(), 1, None, 0, 1, 0, 0, s, mask.data_ptr(), None)


def dx():
    return LIB.sp_debug_gemm_tf32_async(rows, d, d, dz.data_ptr(), d, 0, W.data_ptr(), d, 0, 5, y.data_ptr(), d,
                                        None, 1, None, d, 1, 0, 0, s, None, mask.data_ptr())


def dw():
    return LIB.sp_debug_gemm_tf32_async(d, d, rows, x.data_ptr(), d, 1, dz.data_ptr(), d, 1, 3, parts.data_ptr(), d,
                                        None, 0, None, 0, splits, bn.value, cta.value, s, None, None)


def timed(fn, reps=20):
    for _ in range(3):
        rc = fn()
        assert not rc, rc
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


flop = 2.0 * rows * d * d
out = {"shape": [rows, d], "dw_choice": {"splits": splits, "cta": cta.value, "block_n": bn.value}}
for name, fn in (("fwd", fwd), ("dx", dx), ("dw", dw)):
    ms = timed(fn)
    out[name] = {"us": ms * 1e3, "tflops": flop / ms / 1e9}
torch.backends.cuda.matmul.allow_tf32 = True
out["cublas_tf32_xW"] = {"us": timed(lambda: (torch.matmul(x, W, out=y), 0)[1]) * 1e3}
out["cublas_tf32_xW"]["tflops"] = flop / out["cublas_tf32_xW"]["us"] / 1e6
out["cublas_tf32_xTdz"] = {"us": timed(lambda: (torch.matmul(x.t(), dz), 0)[1]) * 1e3}
out["cublas_tf32_xTdz"]["tflops"] = flop / out["cublas_tf32_xTdz"]["us"] / 1e6
print(json.dumps(out))
