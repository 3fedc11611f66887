"""Do a small pinned H2D copy and a small tcgen05 GEMM slow each other down when they run
concurrently on two streams? Times each alone and both together (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

LIB = _capi.LIB
rows, d = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (4096, 768)))
nbytes = d * d * 2 + d * 4
h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
dv = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
x = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
W = torch.randn(d, d, device="cuda").to(torch.bfloat16)
bias = torch.randn(d, device="cuda")
o = torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)
s_copy, s_comp = torch.cuda.Stream(), torch.cuda.Stream()
N = 50


def gemm():
    assert LIB.sp_debug_gemm_bf16_async(rows, d, d, x.data_ptr(), d, 0, W.data_ptr(), d, 1, 0, o.data_ptr(), d,
                                        bias.data_ptr(), 1, None, 0, 1, 0, 0, s_comp.cuda_stream) == 0


def timed(copy, comp):
    torch.cuda.synchronize()
    ec = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    eg = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ec[0].record(s_copy)
    eg[0].record(s_comp)
    for _ in range(N):
        if copy:
            with torch.cuda.stream(s_copy):
                dv.copy_(h, non_blocking=True)
        if comp:
            gemm()
    ec[1].record(s_copy)
    eg[1].record(s_comp)
    torch.cuda.synchronize()
    return ec[0].elapsed_time(ec[1]) * 1e3 / N, eg[0].elapsed_time(eg[1]) * 1e3 / N


for _ in range(2):
    timed(True, True)
c_alone, _ = timed(True, False)
_, g_alone = timed(False, True)
c_both, g_both = timed(True, True)
print(f"copy {nbytes/1e6:.2f} MB: alone {c_alone:.1f} us ({nbytes/c_alone/1e3:.1f} GB/s), with GEMM {c_both:.1f} us")
print(f"GEMM {rows}x{d}x{d}: alone {g_alone:.1f} us, with copies {g_both:.1f} us")
