"""Superpipeline training step (run_train_step path, bf16 tcgen05) on the BASELINE training
configs with the reference's square dense blocks:
  c2   48 x d=1600, 16384 rows, SP(4,2)             (GPT-2 XL depth/width; the bench.py headline)
  c4   32 x d=1280, 65792 rows (256 x 257), SP(4,2)  (ViT-H/14 depth/width), activations saved
       on device (ckpt off) and offloaded to pinned host memory (ckpt on)
Inputs are device-resident (train_step_device); weights stream from the executor's pinned host
master every step. Prints one JSON line per run: samples/s, ms/step, per-layer roofline
(max of FLOPs at the measured bf16 peak and host-link bytes at the measured pinned bandwidth;
activation offload adds its D2H in the forward and its H2D in the backward), HBM peaks."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import bench  # noqa: E402
import torch  # noqa: E402

import paper_2410_08791_b200 as sp  # noqa: E402
from infer_bench import build_weights  # noqa: E402

CONFIGS = {
    "c2": dict(n=48, d=1600, rows=16384, windows=[(4, 2)], ckpt=[False, True]),
    "c4": dict(n=32, d=1280, rows=65792, windows=[(4, 2)], ckpt=[False, True]),
}


def link_ms(a, b, link):
    """Time to move a bytes H2D and b bytes D2H concurrently: each direction at its simplex
    rate, and both together at most 2 x the measured per-direction duplex rate."""
    h2d, d2h, dup = (link[k] * 1e9 for k in ("h2d_gbs", "d2h_gbs", "duplex_gbs_per_dir"))
    return max(a / h2d, b / d2h, (a + b) / (2 * dup))


def roofline_ms(n, d, rows, ckpt, link, peak, slots):
    """Ring lower bound (bench.layer_roofline, plus activation offload): S slots carry at
    most S layers across each direction reversal, so forward and backward each load >= n - S
    layers; every layer writes back; with offload each forward layer's input goes D2H and
    comes back H2D in the backward."""
    S = min(slots, n)
    lb = (d * d + d) * 4           # fp32 master per layer, each direction
    act = rows * d * 2             # bf16 saved activation per layer
    fwd_flop, bwd_flop = 2.0 * rows * d * d / peak, 4.0 * rows * d * d / peak
    t = 0.0
    for L in range(n):             # forward: the first S layers are still resident
        t += max(fwd_flop, link_ms(lb if L >= S else 0, act if ckpt else 0, link))
    for pos in range(n):           # backward, layer n-1 first (layer 0 needs no dX)
        fl = fwd_flop if pos == n - 1 else bwd_flop
        t += max(fl, link_ms((lb if pos >= S else 0) + (act if ckpt else 0), lb, link))
    return 1e3 * t


def cpu_reference_rate(d, rows_total, n_layers, sample_rows=64):
    """the reference's reference_train_step (oracle/_ref) on one host core, timed on a
    one-layer model over `sample_rows` rows, extrapolated linearly in rows and layers."""
    import time
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Reference
    ref = Reference()
    W, b, _ = ref.build_model(7, 1, d)
    rows = min(sample_rows, rows_total)
    x, t = ref.make_input(7, 0, rows, d), ref.make_input(7, 1, rows, d)
    t0 = time.perf_counter()
    ref.train_step(W, b, x, t, 0.01)
    dt = time.perf_counter() - t0
    full = dt * (rows_total / rows) * n_layers
    return rows_total / full, (f"reference_train_step, 1 core, 1 of {n_layers} layers x {rows} of "
                               f"{rows_total} rows ({dt:.2f} s), extrapolated linearly")


def main():
    p = argparse.ArgumentParser()
    p.add_argument("configs", nargs="*", default=["c4"])
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--lr", type=float, default=0.01)
    p.add_argument("--cpu-baseline", action="store_true",
                   help="also time the reference's CPU train step per config (one layer, extrapolated)")
    a = p.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops_sustained"] * 1e12
    link = bench.measure_link(torch, chunk=(1280 * 1280 + 1280) * 4)
    print(json.dumps({"link": link}), flush=True)
    for name in a.configs:
        c = CONFIGS[name]
        n, d, rows = c["n"], c["d"], c["rows"]
        weights = build_weights(n, d)
        x = torch.from_numpy(sp.make_input(7, 0, rows, d)).cuda()
        t = torch.from_numpy(sp.make_input(7, 1, rows, d)).cuda()
        for k, kp in c["windows"]:
            for ckpt in c["ckpt"]:
                ex = sp.Executor(n, d, sp.StrategyConfig(sp.SUPERPIPELINE, k, kp),
                                 numerics=sp.BF16, checkpointing=ckpt, trace=0)
                for i, (W, b) in enumerate(weights):
                    ex.register_layer(i, W, b)
                for _ in range(3):
                    ex.train_step_ptr(x.data_ptr(), t.data_ptr(), rows, a.lr, device=True)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.steps):
                    loss = ex.train_step_ptr(x.data_ptr(), t.data_ptr(), rows, a.lr, device=True)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / a.steps
                st = ex.stats()
                roof = roofline_ms(n, d, rows, ckpt, link, peak, st["n_slots"])
                print(json.dumps({
                    "config": name, "layers": n, "d": d, "rows": rows, "k": k, "k_prime": kp,
                    "checkpointing": ckpt, "ms_per_step": ms, "samples_per_s": rows / ms * 1e3,
                    "roofline_ms": roof, "frac_of_roofline": roof / ms, "loss": loss,
                    "h2d_gb": st["h2d_bytes"] / 1e9, "d2h_gb": st["d2h_bytes"] / 1e9,
                    "ledger_peak_gb": st["peak_bytes"] / 1e9,
                    "ledger_weights_gb": st["peak_weight_bytes"] / 1e9,
                    "ledger_acts_gb": st["peak_activation_bytes"] / 1e9,
                    "hbm_reserved_gb": st["hbm_reserved_bytes"] / 1e9,
                    "graph_replays": st["graph_replays"]}), flush=True)
                ex.close()
        if a.cpu_baseline:
            rate, how = cpu_reference_rate(d, rows, n)
            print(json.dumps({"config": name, "cpu_baseline": {"value": rate, "unit": "samples/s", "cores": 1,
                                                               "kind": "reference", "sample": how}}), flush=True)


if __name__ == "__main__":
    main()
