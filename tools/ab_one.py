"""One GEMM launch (shape/kind from argv) through a given libsuperpipe build, for ncu capture.
Usage: python tools/ab_one.py LIB.so rows d fwd|dx|dw"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

LIB = _capi.load(os.path.abspath(sys.argv[1]))
rows, d, kind = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
x = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
dz = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
W = torch.randn(d, d, device="cuda").to(torch.bfloat16)
bias = torch.randn(d, device="cuda")
out = torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)
splits = int(_capi.LIB.sp_debug_dw_splits(d, rows))
parts = torch.empty(splits * d * d, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    if kind == "fwd":
        rc = LIB.sp_debug_gemm_bf16_async(rows, d, d, x.data_ptr(), d, 0, W.data_ptr(), d, 1, 0,
                                          out.data_ptr(), d, bias.data_ptr(), 1, None, 0, 1, 0, 0, st)
    elif kind == "dx":
        rc = LIB.sp_debug_gemm_bf16_async(rows, d, d, dz.data_ptr(), d, 0, W.data_ptr(), d, 0, 2,
                                          out.data_ptr(), d, None, 1, x.data_ptr(), d, 1, 0, 0, st)
    else:
        rc = LIB.sp_debug_gemm_bf16_async(d, d, rows, x.data_ptr(), d, 1, dz.data_ptr(), d, 1, 3,
                                          parts.data_ptr(), d, None, 0, None, 0, splits, 0, 0, st)
    assert rc == 0
torch.cuda.synchronize()
