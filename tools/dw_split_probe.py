"""dW = x^T dz split-K sweep: (variant, splits) -> device time of the fp32-partials GEMM, warm,
back to back (CUDA events), min of 3 interleaved rounds. Usage: python tools/dw_split_probe.py rows d"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

LIB = _capi.LIB
rows, d = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (16384, 1600)))
x = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
dz = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
parts = torch.empty(16 * d * d, device="cuda")
st = torch.cuda.current_stream().cuda_stream
fl = 2.0 * rows * d * d
res = {}
for rnd in range(3):
    for cta, bn in [(1, 192), (1, 256), (2, 256)]:
        for s in range(1, 11):
            fn = lambda: LIB.sp_debug_gemm_bf16_async(d, d, rows, x.data_ptr(), d, 1, dz.data_ptr(), d, 1, 3,
                                                       parts.data_ptr(), d, None, 0, None, 0, s, bn, cta, st)
            if fn() != 0:
                continue
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                fn()
            e1.record()
            e1.synchronize()
            k = (cta, bn, int(LIB.sp_debug_effective_splits(rows, s)))
            res[k] = min(res.get(k, 1e9), e0.elapsed_time(e1) / 10 * 1e3)
for (cta, bn, s), us in sorted(res.items()):
    print(json.dumps({"cta": cta, "bn": bn, "splits": s, "us": round(us, 1),
                      "tflops": round(fl / us / 1e6, 1)}))
print(json.dumps({"auto_splits": int(LIB.sp_debug_dw_splits(d, rows))}))
