"""Pinned host<->device bandwidth vs the number of concurrent copy streams per direction (does
splitting copies across copy engines raise PCIe throughput?). 256 MB per direction per rep,
split evenly over the streams; H2D alone, D2H alone, and both at once."""
import json
import torch

MB = 1 << 20
n = 256 * MB
h_src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_dst = torch.empty(n, dtype=torch.uint8, device="cuda")
d_src = torch.empty(n, dtype=torch.uint8, device="cuda")


def run(k, h2d, d2h, chunk_mb=None, reps=8):
    up = [torch.cuda.Stream() for _ in range(k)]
    dn = [torch.cuda.Stream() for _ in range(k)]
    part = n // k
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in up + dn:
        s.wait_event(e0)
    for _ in range(reps):
        for i in range(k):
            sl = slice(i * part, (i + 1) * part)
            if h2d:
                with torch.cuda.stream(up[i]):
                    d_dst[sl].copy_(h_src[sl], non_blocking=True)
            if d2h:
                with torch.cuda.stream(dn[i]):
                    h_dst[sl].copy_(d_src[sl], non_blocking=True)
    cur = torch.cuda.current_stream()
    for s in up + dn:
        ev = torch.cuda.Event()
        ev.record(s)
        cur.wait_event(ev)
    e1.record()
    e1.synchronize()
    return n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9


run(2, True, True, reps=2)
for k in (1, 2, 4):
    print(json.dumps({"streams_per_dir": k, "h2d_gbs": round(run(k, True, False), 1),
                      "d2h_gbs": round(run(k, False, True), 1),
                      "duplex_gbs_per_dir": round(run(k, True, True), 1)}))
