"""Llama-3-8B layer GEMMs at C3's 32 x 2048 tokens: our tcgen05 kernels with the epilogues the
block uses (SwiGLU gate/up, residual down / Wo, QKV) against a plain bf16 store and torch.matmul
(cuBLAS, context only), with the median SM clock and board power over a ~0.4 s back-to-back run
(NVML), timed over that same run: under the 1000 W cap the clock a kernel holds decides its rate.
Usage: python tools/llama_gemm_probe.py [G ...]   (CTA-pair rasterisation groups to try, debug knob "raster")"""
import ctypes as C
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

LIB = _capi.LIB
BIAS_BF16, RESID_F32, SWIGLU = 0, 6, 9
T, D, FF, Q = 32 * 2048, 4096, 14336, 6144
st = torch.cuda.current_stream().cuda_stream
import pynvml  # noqa: E402

pynvml.nvmlInit()
NVH = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    clk, pw, stop = [], [], [False]

    def sample():
        while not stop[0]:
            clk.append(pynvml.nvmlDeviceGetClockInfo(NVH, pynvml.NVML_CLOCK_SM))
            pw.append(pynvml.nvmlDeviceGetPowerUsage(NVH) / 1e3)
            time.sleep(0.01)
    th = threading.Thread(target=sample)
    th.start()
    n = max(1, int(1.5e6 / us))
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    stop[0] = True
    th.join()
    return e0.elapsed_time(e1) / n * 1e3, sorted(clk)[len(clk) // 2], sorted(pw)[len(pw) // 2]


def report(name, M, N, K, fn):
    us, mhz, w = timeit(fn)
    tf = 2.0 * M * N * K / us / 1e6
    print(json.dumps({"case": name, "M": M, "N": N, "K": K, "us": round(us, 1), "tflops": round(tf, 1),
                      "sm_mhz": mhz, "watts": round(w), "tflops_per_ghz": round(tf / mhz * 1e3, 1)}), flush=True)


def ours(name, M, N, K, A, lda, B, ldb, epi, out, ldo, gate=None, ldg=0, aux=None, ldaux=0):
    args = _capi.GemmArgs(M, N, K, A.data_ptr(), lda, 0, B.data_ptr(), ldb, 1, epi, out.data_ptr(), ldo,
                          None, 0, gate.data_ptr() if gate is not None else None, ldg, 1, 0, 0,
                          aux.data_ptr() if aux is not None else None, ldaux, 0, st)

    def f():
        assert LIB.sp_debug_gemm_ex(C.byref(args)) == 0
    report(name, M, N, K, f)


bf = torch.bfloat16
x = torch.randn(T, D, device="cuda").to(bf)
W13 = (torch.randn(D, 2 * FF, device="cuda") * 0.02).to(bf)
g = torch.empty(T, FF, device="cuda", dtype=bf)
W2 = (torch.randn(FF, D, device="cuda") * 0.02).to(bf)
res = torch.randn(T, D, device="cuda")
y = torch.empty(T, D, device="cuda")
Wq = (torch.randn(D, Q, device="cuda") * 0.02).to(bf)
qkv = torch.empty(T, Q, device="cuda", dtype=bf)
for G in [int(v) for v in sys.argv[1:]] or [8]:
    assert LIB.sp_debug_set(None, b"raster", G) == 0
    print(json.dumps({"raster_group": G}))
    ours("gate_up_swiglu", T, 2 * FF, D, x, D, W13, 2 * FF, SWIGLU, g, FF)
    ours("down_resid", T, D, FF, g, FF, W2, D, RESID_F32, y, D, gate=res, ldg=D)
    ours("qkv_bf16", T, Q, D, x, D, Wq, Q, BIAS_BF16, qkv, Q)
report("cublas_gate_up", T, 2 * FF, D, lambda: torch.matmul(x, W13))
report("cublas_down", T, D, FF, lambda: torch.matmul(g, W2))
report("cublas_qkv", T, Q, D, lambda: torch.matmul(x, Wq))
