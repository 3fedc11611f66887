"""Inside a CUDA graph, does a kernel that depends on the FIRST of a chain of D2H memcpy nodes
start after that copy, or only after the whole chain? Captures: stream A = 24 x 10 MB D2H
copies (event after the first); stream B = waits that event, then a short kernel; replays and
reports when B's kernel ran relative to A's copies (CUDA events). Eager enqueue for contrast.
Usage: python tools/graph_memcpy_probe.py"""
import json

import torch

N, MB = 24, 10 << 20
dev = torch.empty(N * MB, dtype=torch.uint8, device="cuda")
host = torch.empty(N * MB, dtype=torch.uint8, pin_memory=True)
x = torch.zeros(1 << 20, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
first = torch.cuda.Event()
t0, t_first, t_all, t_k = (torch.cuda.Event(enable_timing=True, external=True) for _ in range(4))


def body():
    t0.record(sa)
    sb.wait_stream(sa)
    with torch.cuda.stream(sa):
        for i in range(N):
            host[i * MB:(i + 1) * MB].copy_(dev[i * MB:(i + 1) * MB], non_blocking=True)
            if i == 0:
                t_first.record(sa)
                first.record(sa)
        t_all.record(sa)
    with torch.cuda.stream(sb):
        sb.wait_event(first)
        x.add_(1.0)
        t_k.record(sb)
    sa.wait_stream(sb)


def times():
    torch.cuda.synchronize()
    return {"first_copy_done_ms": t0.elapsed_time(t_first), "all_copies_done_ms": t0.elapsed_time(t_all),
            "kernel_done_ms": t0.elapsed_time(t_k)}


body()
eager = times()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=sa):
    body()
for _ in range(2):
    g.replay()
graph = times()
print(json.dumps({"eager": eager, "graph": graph}))
