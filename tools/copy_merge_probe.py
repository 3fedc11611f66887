"""Would merging a 2-layer H2D group into one copy pay? Pinned H2D throughput of 2 x 10.24 MB
copies vs 1 x 20.48 MB per group, alone and under a concurrent D2H stream (duplex)."""
import json
import torch

LB = (1600 * 1600 + 1600) * 4
groups = 24
h = torch.empty(2 * LB * groups, dtype=torch.uint8, pin_memory=True)
dv = torch.empty(2 * LB * groups, dtype=torch.uint8, device="cuda")
hd = torch.empty(2 * LB * groups, dtype=torch.uint8, pin_memory=True)
ds = torch.empty(2 * LB * groups, dtype=torch.uint8, device="cuda")
s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()


def run(merged, duplex):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_up)
    s_dn.wait_event(e0)
    with torch.cuda.stream(s_up):
        for g in range(groups):
            base = 2 * LB * g
            if merged:
                dv[base:base + 2 * LB].copy_(h[base:base + 2 * LB], non_blocking=True)
            else:
                dv[base:base + LB].copy_(h[base:base + LB], non_blocking=True)
                dv[base + LB:base + 2 * LB].copy_(h[base + LB:base + 2 * LB], non_blocking=True)
    if duplex:
        with torch.cuda.stream(s_dn):
            for g in range(2 * groups):
                hd[LB * g:LB * (g + 1)].copy_(ds[LB * g:LB * (g + 1)], non_blocking=True)
    e1.record(s_up)
    e1.synchronize()
    return 2 * LB * groups / (e0.elapsed_time(e1) * 1e-3) / 1e9


run(True, True)
for duplex in (False, True):
    best = {m: max(run(m, duplex) for _ in range(4)) for m in (False, True)}
    print(json.dumps({"duplex": duplex, "2x10MB_gbs": round(best[False], 1), "1x20MB_gbs": round(best[True], 1)}))
