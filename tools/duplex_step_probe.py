"""Per-direction PCIe throughput for the backward's copy pattern: 42 layer images (10.25 MB)
H2D on one stream while 42 go D2H on another, alone and with the step's GEMMs running
concurrently on a third stream (does tensor-core / HBM load slow the copy engines?).
Usage: python tools/duplex_step_probe.py"""
import json

import torch

LB = (1600 * 1600 + 1600) * 4
N = 42
h_up = torch.empty(N * LB, dtype=torch.uint8, pin_memory=True)
h_dn = torch.empty(N * LB, dtype=torch.uint8, pin_memory=True)
d_up = torch.empty(N * LB, dtype=torch.uint8, device="cuda")
d_dn = torch.empty(N * LB, dtype=torch.uint8, device="cuda")
a = torch.randn(16384, 1600, device="cuda", dtype=torch.bfloat16)
w = torch.randn(1600, 1600, device="cuda", dtype=torch.bfloat16)
o = torch.empty(16384, 1600, device="cuda", dtype=torch.bfloat16)
s_up, s_dn, s_c = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def run(up, dn, gemm, reps=3):
    res = []
    for _ in range(reps):
        torch.cuda.synchronize()
        start = torch.cuda.Event(enable_timing=True)
        start.record()
        ev = {}
        for name, s, on in (("up", s_up, up), ("dn", s_dn, dn)):
            if not on:
                continue
            s.wait_event(start)
            e1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                for i in range(N):
                    if name == "up":
                        d_up[i * LB:(i + 1) * LB].copy_(h_up[i * LB:(i + 1) * LB], non_blocking=True)
                    else:
                        h_dn[i * LB:(i + 1) * LB].copy_(d_dn[i * LB:(i + 1) * LB], non_blocking=True)
                e1.record(s)
            ev[name] = e1
        if gemm:
            s_c.wait_event(start)
            with torch.cuda.stream(s_c):
                for _ in range(160):
                    torch.mm(a, w, out=o)
        torch.cuda.synchronize()
        res.append({k: N * LB / (start.elapsed_time(e) * 1e-3) / 1e9 for k, e in ev.items()})
    return {k: max(r[k] for r in res) for k in res[0]}


out = {"h2d_alone": run(True, False, False), "d2h_alone": run(False, True, False),
       "duplex": run(True, True, False), "h2d_with_gemm": run(True, False, True),
       "duplex_with_gemm": run(True, True, True)}
print(json.dumps(out))

# Same pattern with host buffers from the executor's own allocator (sp_host_alloc:
# cudaHostAllocPortable, first touched by this thread), to separate allocation / NUMA
# placement effects from the executor's scheduling.
import os  # noqa: E402
import sys  # noqa: E402

import numpy as np  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_08791_b200 as sp  # noqa: E402

hb_up = sp.HostBuffer((N * LB,), np.uint8)
hb_dn = sp.HostBuffer((N * LB,), np.uint8)
hb_up.array[:] = 1
hb_dn.array[:] = 1
h_up = torch.from_numpy(hb_up.array)
h_dn = torch.from_numpy(hb_dn.array)
print(json.dumps({"sp_host_alloc": {"h2d_alone": run(True, False, False), "duplex": run(True, True, False)}}))
