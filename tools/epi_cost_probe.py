"""Cost of the fused epilogues at the GPT-2 XL block's GEMM shapes (16 x 1024 tokens): the same
mainloop with each epilogue the block uses, against a plain fp32 / bf16 store and torch.matmul
(cuBLAS, context only). Back-to-back launches between CUDA events. Prints one JSON line per case.
Usage: python tools/epi_cost_probe.py [vit]   (vit: ViT-H/14 at 256 x 257 tokens, exact-erf GELU)"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

LIB = _capi.LIB
BIAS_BF16, GATE_BF16, F32, RESID_F32, GELU_BF16, GELU_GATE_BF16 = 0, 2, 3, 6, 7, 8
VIT = len(sys.argv) > 1 and sys.argv[1] == "vit"
T, D, FF, Q = (65792, 1280, 5120, 3840) if VIT else (16384, 1600, 6400, 4800)
ACT = 1 if VIT else 0  # GELU_ERF / GELU_TANH
st = torch.cuda.current_stream().cuda_stream


try:
    import pynvml
    pynvml.nvmlInit()
    NVH = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
except Exception:  # noqa: BLE001
    NVH = None
CLK = {}


def timeit(fn, reps=20):
    """us per launch; also the median SM clock / power over a ~0.4 s back-to-back run (NVML),
    because these kernels run into the board's power cap and their clock depends on the epilogue."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    if NVH is not None:
        import threading
        import time
        clk, pw, stop = [], [], [False]

        def sample():
            while not stop[0]:
                clk.append(pynvml.nvmlDeviceGetClockInfo(NVH, pynvml.NVML_CLOCK_SM))
                pw.append(pynvml.nvmlDeviceGetPowerUsage(NVH) / 1e3)
                time.sleep(0.01)
        n = max(1, int(4e5 / us))
        th = threading.Thread(target=sample)
        th.start()
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
        stop[0] = True
        th.join()
        CLK["sm_mhz"] = sorted(clk)[len(clk) // 2] if clk else None
        CLK["watts"] = sorted(pw)[len(pw) // 2] if pw else None
    return us


def run(name, M, N, K, A, lda, a_mn, B, ldb, b_mn, epi, out, ldo, bias=None, gate=None, ldg=0, aux=None, ldaux=0):
    args = _capi.GemmArgs(M, N, K, A.data_ptr(), lda, a_mn, B.data_ptr(), ldb, b_mn, epi, out.data_ptr(), ldo,
                          bias.data_ptr() if bias is not None else None, 0,
                          gate.data_ptr() if gate is not None else None, ldg, 1, 0, 0,
                          aux.data_ptr() if aux is not None else None, ldaux, ACT, st)

    def f():
        rc = LIB.sp_debug_gemm_ex(C.byref(args))
        assert rc == 0, rc
    us = timeit(f)
    print(json.dumps({"case": name, "M": M, "N": N, "K": K, "us": round(us, 1),
                      "tflops": round(2.0 * M * N * K / us / 1e6, 1), **CLK}), flush=True)


bf = torch.bfloat16
x = torch.randn(T, D, device="cuda").to(bf)
g = torch.randn(T, FF, device="cuda").to(bf)
W1 = (torch.randn(D, FF, device="cuda") * 0.02).to(bf)
W2 = (torch.randn(FF, D, device="cuda") * 0.02).to(bf)
b1 = torch.randn(FF, device="cuda")
b2 = torch.randn(D, device="cuda")
out16 = torch.empty(T, FF, device="cuda", dtype=bf)
aux16 = torch.empty(T, FF, device="cuda", dtype=bf)
out32 = torch.empty(T, FF, device="cuda")
res = torch.randn(T, D, device="cuda")
y32 = torch.empty(T, D, device="cuda")
# FC1: x W1 (+b1) -> GELU (out + pre-activation) vs bias-only bf16 vs fp32
run("fc1_gelu", T, FF, D, x, D, 0, W1, FF, 1, GELU_BF16, out16, FF, bias=b1, aux=aux16, ldaux=FF)
run("fc1_bias_bf16", T, FF, D, x, D, 0, W1, FF, 1, BIAS_BF16, out16, FF, bias=b1)
run("fc1_f32", T, FF, D, x, D, 0, W1, FF, 1, F32, out32, FF)
# dg = dy W2^T * gelu'(h) (K-major B) vs a plain bf16 / fp32 store
dy = torch.randn(T, D, device="cuda").to(bf)
run("dg_gelu_gate", T, FF, D, dy, D, 0, W2, D, 0, GELU_GATE_BF16, out16, FF, gate=aux16, ldg=FF)
run("dg_gate_bf16", T, FF, D, dy, D, 0, W2, D, 0, GATE_BF16, out16, FF)
run("dg_f32", T, FF, D, dy, D, 0, W2, D, 0, F32, out32, FF)
# FC2: g W2 + b2 + residual (fp32) vs plain fp32
run("fc2_resid", T, D, FF, g, FF, 0, W2, D, 1, RESID_F32, y32, D, bias=b2, gate=res, ldg=D)
run("fc2_f32", T, D, FF, g, FF, 0, W2, D, 1, F32, y32, D)
for name, a, b in (("cublas_fc1", x, W1), ("cublas_fc2", g, W2)):
    us = timeit(lambda: torch.matmul(a, b))
    print(json.dumps({"case": name, "us": round(us, 1),
                      "tflops": round(2.0 * a.shape[0] * a.shape[1] * b.shape[1] / us / 1e6, 1), **CLK}))
