"""Launch-to-launch cost of the tcgen05 GEMM inside a CUDA graph: a chain of n dependent GEMM
launches (ping-pong activations) captured once and replayed; reports us per GEMM node vs the
kernel's own duration (ncu: ~12.9 us at 4096 x 768 x 768)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_08791_b200 import _capi  # noqa: E402

LIB = _capi.LIB
rows, d, n = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 768, 12)))
with_copies = len(sys.argv) > 4 and sys.argv[4] == "copies"  # a concurrent H2D chain in the graph
nbytes = d * d * 2 + d * 4
h = torch.empty(nbytes * n, dtype=torch.uint8, pin_memory=True)
dv = torch.empty(nbytes * n, dtype=torch.uint8, device="cuda")
s2 = torch.cuda.Stream()
a = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
b = torch.empty_like(a)
W = (torch.randn(d, d, device="cuda") * 0.03).to(torch.bfloat16)
bias = torch.zeros(d, device="cuda")
s = torch.cuda.Stream()


def chain(st):
    if with_copies:  # fork a copy chain (one layer image per GEMM) onto s2, joined at the end
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        s2.wait_event(ev)
        with torch.cuda.stream(s2):
            for i in range(n):
                dv[i * nbytes:(i + 1) * nbytes].copy_(h[i * nbytes:(i + 1) * nbytes], non_blocking=True)
    src, dst = a, b
    for _ in range(n):
        assert LIB.sp_debug_gemm_bf16_async(rows, d, d, src.data_ptr(), d, 0, W.data_ptr(), d, 1, 0,
                                            dst.data_ptr(), d, bias.data_ptr(), 1, None, 0, 1, 0, 0, st) == 0
        src, dst = dst, src
    if with_copies:
        ev2 = torch.cuda.Event()
        ev2.record(s2)
        torch.cuda.current_stream().wait_event(ev2)


with torch.cuda.stream(s):
    chain(s.cuda_stream)  # warm (tensor maps, attributes)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    chain(s.cuda_stream)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record()
for _ in range(reps):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"graph chain of {n} GEMMs {rows}x{d}x{d}{' + concurrent H2D chain' if with_copies else ''}: "
      f"{e0.elapsed_time(e1) * 1e3 / reps / n:.1f} us per GEMM node")
if with_copies:  # the copy chain alone, for reference
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2, stream=s):
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        s2.wait_event(ev)
        with torch.cuda.stream(s2):
            for i in range(n):
                dv[i * nbytes:(i + 1) * nbytes].copy_(h[i * nbytes:(i + 1) * nbytes], non_blocking=True)
        ev2 = torch.cuda.Event()
        ev2.record(s2)
        torch.cuda.current_stream().wait_event(ev2)
    for _ in range(3):
        g2.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        g2.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"  copy chain alone: {e0.elapsed_time(e1) * 1e3 / reps / n:.1f} us per {nbytes / 1e6:.2f} MB copy")
