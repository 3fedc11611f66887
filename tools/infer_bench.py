"""Superpipeline inference (run_inference path, bf16 tcgen05) on the BASELINE inference
configs with the reference's square dense blocks:
  c1   12 x d=768,  4 items x 1 row,  SP(2,1)         (configs[0] shape, latency-bound)
  c1b  12 x d=768,  1 item x 4096 rows, SP(2,1)
  c3   32 x d=4096, 1 item x 65536 rows (32 x 2048), SP(4,2)   (Llama-3-8B depth/width)
  c5   80 x d=8192, 1 item x 8192 rows, SP(8,k') sweep, capacity 40 GB (Llama-3-70B depth/width)
Weights: build_model(7, n, d) (splitmix64, generated in parallel threads); bf16 on the wire.
Prints one JSON line per run: samples/s (rows/s), ms/call, per-layer roofline, HBM."""
import argparse
import json
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2410_08791_b200 as sp  # noqa: E402
from paper_2410_08791_b200 import _capi  # noqa: E402

CONFIGS = {
    "c1": dict(n=12, d=768, items=4, rows=1, windows=[(2, 1)]),
    # c1 with sp_set_item_batching: the 4 items stream the layer stack once (layer-major)
    "c1x": dict(n=12, d=768, items=4, rows=1, windows=[(2, 1)], batching=True),
    "c1b": dict(n=12, d=768, items=1, rows=4096, windows=[(2, 1), (4, 2)]),
    "c3": dict(n=32, d=4096, items=1, rows=65536, windows=[(4, 2)]),
    "c5": dict(n=80, d=8192, items=1, rows=8192, windows=[(8, 1), (8, 2), (8, 4), (12, 6)],
               capacity=40 << 30),
}


def build_weights(n, d, threads=16):
    out = [None] * n

    def work(lo):
        for i in range(lo, n, threads):
            W = np.empty((d, d), np.float32)
            b = np.empty((d,), np.float32)
            _capi.LIB.sp_build_layer(7, i, d, 0, 0, W.ctypes.data, b.ctypes.data)
            out[i] = (W, b)

    th = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return out


def cpu_reference_rate(d, rows_total, n_layers, sample_rows=64):
    """the reference's reference_forward (oracle/_ref, built from its sources) on one
    host core, timed on ONE d-wide layer over `sample_rows` rows and extrapolated linearly in
    rows and layers (every block costs the same). Returns (rows/s, description)."""
    import time
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Reference
    ref = Reference()
    W, b, _ = ref.build_model(7, 1, d)
    rows = min(sample_rows, rows_total)
    x = ref.make_input(7, 0, rows, d)
    t0 = time.perf_counter()
    ref.forward(W, b, x)
    dt = time.perf_counter() - t0
    full = dt * (rows_total / rows) * n_layers
    return rows_total / full, (f"reference_forward, 1 core, 1 of {n_layers} layers x {rows} of {rows_total} rows "
                               f"({dt:.2f} s), extrapolated linearly")


def main():
    p = argparse.ArgumentParser()
    p.add_argument("configs", nargs="*", default=["c1", "c1b", "c3"])
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--mode", default="batch", choices=["batch", "sequential"])
    p.add_argument("--cpu-baseline", action="store_true",
                   help="also time the reference's CPU forward per config (one layer, extrapolated)")
    p.add_argument("--reference-prefetch", action="store_true",
                   help="copies wait for the reference policy's trigger compute (no eager prefetch)")
    a = p.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops_sustained"] * 1e12

    def copy_rate(nbytes, reps=40):
        """Measured pinned host -> HBM rate for back-to-back copies of one layer's size (the rate a
        small-layer config such as C1 can reach: per-copy latency dominates below a few MB)."""
        src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        for _ in range(5):
            dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        return nbytes * reps / (e0.elapsed_time(e1) * 1e-3)

    for name in a.configs:
        c = CONFIGS[name]
        n, d, items, rows = c["n"], c["d"], c["items"], c["rows"]
        weights = build_weights(n, d)
        x = torch.from_numpy(np.stack([sp.make_input(7, i, rows, d) for i in range(items)])).cuda()
        y = torch.empty_like(x)
        for k, kp in c["windows"]:
            tmode = sp.BATCH if a.mode == "batch" else sp.SEQUENTIAL
            ex = sp.Executor(n, d, sp.StrategyConfig(sp.SUPERPIPELINE, k, kp, tmode), numerics=sp.BF16,
                             trace=0, capacity_bytes=c.get("capacity", 0))
            for i, (W, b) in enumerate(weights):
                ex.register_layer(i, W, b)
            ex.set_item_batching(c.get("batching", False))
            ex.set_eager_prefetch(not a.reference_prefetch)
            for _ in range(2):
                ex.forward_ptr(x.data_ptr(), rows, items, y.data_ptr(), device=True)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                ex.forward_ptr(x.data_ptr(), rows, items, y.data_ptr(), device=True)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            st = ex.stats()
            wire = d * d * 2 + d * 4
            passes = 1 if c.get("batching") else items  # layer-stack passes over the link
            roof = passes * n * max(2.0 * rows * d * d * items / passes / peak, wire / 55.5e9) * 1e3
            small = copy_rate(wire)  # this layer size's achievable link rate
            roof_small = passes * n * max(2.0 * rows * d * d * items / passes / peak, wire / small) * 1e3
            print(json.dumps({
                "config": name, "layers": n, "d": d, "items": items, "rows": rows, "k": k,
                "item_batching": bool(c.get("batching")), "eager_prefetch": not a.reference_prefetch,
                "transfer_mode": a.mode,
                "k_prime": kp, "ms_per_call": ms, "samples_per_s": items * rows / (ms * 1e-3),
                "layer_roofline_ms": roof, "frac_of_roofline": roof / ms,
                "layer_copy_gbs": small / 1e9, "small_copy_roofline_ms": roof_small,
                "frac_of_small_copy_roofline": roof_small / ms, "host_enqueue_ms": st["host_enqueue_ms"],
                "n_slots": st["n_slots"], "peak_weight_gb": st["peak_weight_bytes"] / 1e9,
                "hbm_reserved_gb": st["hbm_reserved_bytes"] / 1e9,
                "full_residency_bf16_gb": n * wire / 1e9,
                "h2d_gb_per_call": st["h2d_bytes"] / 1e9}), flush=True)
            ex.close()
        if a.cpu_baseline:
            rate, how = cpu_reference_rate(d, items * rows, n)
            print(json.dumps({"config": name, "cpu_baseline": {"value": rate, "unit": "samples/s",
                                                               "cores": 1, "kind": "reference",
                                                               "sample": how}}), flush=True)


if __name__ == "__main__":
    main()
