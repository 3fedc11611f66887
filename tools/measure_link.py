"""Measures the host link (pinned cudaMemcpyAsync) bandwidth the Superpipeline roofline uses:
H2D alone, D2H alone, and both directions concurrently on separate streams (the training
backward overlaps weight prefetch with updated-weight writeback). Prints one JSON line."""
import json
import sys

import torch


def bw(nbytes, reps, fn, streams):
    for s in streams:
        s.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(streams[0])
    for s in streams[1:]:
        s.wait_event(start)
    for _ in range(reps):
        fn()
    for s in streams[1:]:
        ev = torch.cuda.Event()
        ev.record(s)
        streams[0].wait_event(ev)
    end.record(streams[0])
    end.synchronize()
    return nbytes * reps / (start.elapsed_time(end) * 1e-3) / 1e9


def main():
    mb = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    n = mb << 20
    host_a = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    host_b = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    dev_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    dev_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        with torch.cuda.stream(s1):
            dev_a.copy_(host_a, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            host_b.copy_(dev_b, non_blocking=True)

    def both():
        h2d()
        d2h()

    for f in (h2d, d2h, both):
        bw(n, 2, f, [s1, s2])
    res = dict(bytes_per_copy=n, h2d_gbs=bw(n, 10, h2d, [s1, s2]), d2h_gbs=bw(n, 10, d2h, [s1, s2]),
               duplex_gbs_per_dir=bw(n, 10, both, [s1, s2]),
               device=torch.cuda.get_device_name(0))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
