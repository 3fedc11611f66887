"""C1's layer copies are small (1.18 MB bf16 wire image): is a chain of them latency-bound per
copy, and does splitting each layer across two streams (copy engines) help? 12 layer copies:
one stream whole, one stream in halves, two streams in halves, events around the chain.
Usage: python tools/small_copy_probe.py"""
import json

import torch

LB = 768 * 768 * 2 + 768 * 4
N = 12
h = torch.empty(N * LB, dtype=torch.uint8, pin_memory=True)
dv = torch.empty(N * LB, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(mode):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s1)
    s2.wait_event(e0)
    half = LB // 2
    for i in range(N):
        a, b = i * LB, (i + 1) * LB
        if mode == "one_stream_whole":
            with torch.cuda.stream(s1):
                dv[a:b].copy_(h[a:b], non_blocking=True)
        elif mode == "one_stream_halves":
            with torch.cuda.stream(s1):
                dv[a:a + half].copy_(h[a:a + half], non_blocking=True)
                dv[a + half:b].copy_(h[a + half:b], non_blocking=True)
        else:
            with torch.cuda.stream(s1):
                dv[a:a + half].copy_(h[a:a + half], non_blocking=True)
            with torch.cuda.stream(s2):
                dv[a + half:b].copy_(h[a + half:b], non_blocking=True)
    ev = torch.cuda.Event()
    ev.record(s2)
    s1.wait_event(ev)
    e1.record(s1)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / N  # us per layer


out = {}
for m in ("one_stream_whole", "one_stream_halves", "two_streams_halves"):
    for _ in range(3):
        run(m)
    out[m + "_us_per_layer"] = min(run(m) for _ in range(10))
out["gbs_one_stream"] = LB / (out["one_stream_whole_us_per_layer"] * 1e-6) / 1e9
out["gbs_two_streams"] = LB / (out["two_streams_halves_us_per_layer"] * 1e-6) / 1e9
print(json.dumps(out))
