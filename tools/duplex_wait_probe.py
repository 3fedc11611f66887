"""Does gating each copy on a cross-stream event cost PCIe throughput? The backward's duplex
pattern (42 x 10.25 MB H2D in pairs, 42 x 10.25 MB D2H singly) with no waits vs with a
cudaStreamWaitEvent before every op on events recorded (ahead of time) on a third stream by a
short kernel, as the executor's dependency edges do. Usage: python tools/duplex_wait_probe.py"""
import json

import torch

LB = (1600 * 1600 + 1600) * 4
N = 42
h_up = torch.empty(N * LB, dtype=torch.uint8, pin_memory=True)
h_dn = torch.empty(N * LB, dtype=torch.uint8, pin_memory=True)
d_up = torch.empty(N * LB, dtype=torch.uint8, device="cuda")
d_dn = torch.empty(N * LB, dtype=torch.uint8, device="cuda")
s_up, s_dn, s_k = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
dummy = torch.zeros(1024, device="cuda")


def run(wait, gap_us=0.0):
    torch.cuda.synchronize()
    evs = []
    with torch.cuda.stream(s_k):  # the "compute / update" stream: one event per op
        for i in range(N):
            dummy.add_(1.0)
            if gap_us:
                torch.cuda._sleep(int(gap_us * 1900))  # ~1.9 GHz clock cycles
            e = torch.cuda.Event()
            e.record(s_k)
            evs.append(e)
    start = torch.cuda.Event(enable_timing=True)
    start.record()
    s_up.wait_event(start)
    s_dn.wait_event(start)
    with torch.cuda.stream(s_up):
        for i in range(0, N, 2):
            if wait:
                s_up.wait_event(evs[i])
            for j in (i, i + 1):
                d_up[j * LB:(j + 1) * LB].copy_(h_up[j * LB:(j + 1) * LB], non_blocking=True)
    with torch.cuda.stream(s_dn):
        for i in range(N):
            if wait:
                s_dn.wait_event(evs[i])
            h_dn[i * LB:(i + 1) * LB].copy_(d_dn[i * LB:(i + 1) * LB], non_blocking=True)
    e_up, e_dn = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_up.record(s_up)
    e_dn.record(s_dn)
    torch.cuda.synchronize()
    return {"up": N * LB / (start.elapsed_time(e_up) * 1e-3) / 1e9,
            "dn": N * LB / (start.elapsed_time(e_dn) * 1e-3) / 1e9}


for _ in range(2):
    run(False)
out = {"no_waits": max((run(False) for _ in range(3)), key=lambda r: r["up"]),
       "waits_on_done_events": max((run(True) for _ in range(3)), key=lambda r: r["up"])}
print(json.dumps(out))
