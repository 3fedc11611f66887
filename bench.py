#!/usr/bin/env python
"""bench.py — Superpipeline layer-streaming training step on B200 (driver contract).

Workload (BASELINE.json configs[1]): a GPT-2 XL-shape stack — 48
transformer layers at their real shape (d 1600, ff 6400, 25 heads of 64, LayerNorm, GELU,
causal attention; 30.7M parameters per layer, include/superpipe.h "named-shape layers") — one
bf16 training step (forward, the reference's MSE loss, reverse backward + SGD:
reference_train_step semantics, model.cpp:157-184) streamed through a Superpipeline ring
(k=4, k'=2) from pinned host memory. A "step" = one train step over 16 sequences x 1024
tokens of synthetic input (make_input, seed 7); weights: sp_build_block(seed 7). A sample is
one token (one row of the [tokens, d] activations, as the reference's rows).

value: samples (tokens) per second with x/target already in HBM (sp_train_step_device);
e2e:   the same through the host-buffer C-ABI call (sp_train_step): x/target H2D from pinned
       host memory and the loss D2H inside the timed region.
Weights always stream from pinned host memory — that is the path being measured.
--model dense: round 1's stand-in (48 square reference blocks, d=1600).

--impl reference: the reference's own CPU implementation (oracle/_ref, built from the
reference sources) on the host cores: reference_train_step on FLOP-equivalent square blocks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/sec vs peak HBM GB at window k; % of max(FLOP, host-link bytes) roofline"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=15)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--model", default="gpt2-xl", choices=["gpt2-xl", "vit-h14", "llama3-8b", "llama3-70b", "dense"],
                   help="named-shape transformer layers (SURVEY 8(d)) or round 1's square stand-in")
    p.add_argument("--layers", type=int, default=0, help="0 = the model's own layer count")
    p.add_argument("--seqs", type=int, default=16, help="sequences per GPU per step (named shapes)")
    p.add_argument("--seq-len", type=int, default=0, help="0 = the model's own sequence length")
    p.add_argument("--d", type=int, default=1600, help="--model dense: block width")
    p.add_argument("--rows", type=int, default=16384, help="--model dense: batch rows per GPU per step")
    p.add_argument("--k", type=int, default=4)
    p.add_argument("--kp", type=int, default=2)
    p.add_argument("--strategy", default="superpipeline",
                   choices=["superpipeline", "standard", "naive"])
    p.add_argument("--lr", type=float, default=0.01)
    p.add_argument("--ckpt", action="store_true", help="activation offload (the reference's checkpointing)")
    p.add_argument("--infer", action="store_true",
                   help="inference (run_inference) instead of a train step; N > 1 runs N replicas "
                        "(SURVEY 8(e): inference is replicas only, no collective)")
    p.add_argument("--mode", default="batch", choices=["batch", "sequential"],
                   help="TransferMode (sim.hpp:15): one H2D op per k' group, or per layer")
    p.add_argument("--optimizer", default="sgd", choices=["sgd", "adamw"],
                   help="sgd: the reference's update (default); adamw: fp32 m, v in pinned host "
                        "memory streamed with each backward layer, fused AdamW update")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--private-host-copies", action="store_true",
                   help="N>1: one pinned master per rank instead of one per node (shared memory)")
    p.add_argument("--no-variants", action="store_true",
                   help="skip the in-run variants of the same step ('variants')")
    p.add_argument("--sweep", default="", help="comma list of k:kp to report extra lines")
    p.add_argument("--capacity-gb", type=float, default=0.0,
                   help="HBM budget of the ledger (ArenaConfig::capacity_bytes; C5: 40 GB)")
    p.add_argument("--distinct-layers", type=int, default=0,
                   help="--infer: initialise this many distinct layers and register them round-robin "
                        "(0 = every layer distinct; a 70B-shape model's 80 layers take minutes to generate)")
    a = p.parse_args()
    if a.layers == 0:
        a.layers = {"dense": 48, "gpt2-xl": 48, "vit-h14": 32, "llama3-8b": 32, "llama3-70b": 80}[a.model]
    return a


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 8:
                for n, v in zip(names, r[4:8]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def measure_link(torch, mb=256, chunk=10 << 20):
    """Pinned host <-> HBM bandwidth per direction, alone and duplex (both at once). Two copy
    shapes: one 256 MB copy per direction, and trains of `chunk`-byte copies (the ring's
    layer-sized transfers). Each rate reported is the best of three runs of the better of the
    two, so the roofline that divides by it is a bound the executor cannot beat by copy shape."""
    n = mb << 20
    ha = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    hb = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    da = torch.empty(n, dtype=torch.uint8, device="cuda")
    db = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    nc = max(1, min(n // max(chunk, 1), 48))

    def run(h2d, d2h, reps=6, chunked=False):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s1)
        s2.wait_event(e0)
        moved = 0
        for _ in range(reps if not chunked else 2):
            parts = [(i * chunk, (i + 1) * chunk) for i in range(nc)] if chunked else [(0, n)]
            for lo, hi in parts:
                if h2d:
                    with torch.cuda.stream(s1):
                        da[lo:hi].copy_(ha[lo:hi], non_blocking=True)
                if d2h:
                    with torch.cuda.stream(s2):
                        hb[lo:hi].copy_(db[lo:hi], non_blocking=True)
                moved += hi - lo
        ev = torch.cuda.Event()
        ev.record(s2)
        s1.wait_event(ev)
        e1.record(s1)
        e1.synchronize()
        return moved / (e0.elapsed_time(e1) * 1e-3) / 1e9

    run(True, True, 2)
    out = {}
    for key, h, dn in (("h2d_gbs", True, False), ("d2h_gbs", False, True), ("duplex_gbs_per_dir", True, True)):
        # best of three: the bound should use the best rate the box delivers
        big = max(run(h, dn) for _ in range(3))
        small = max(run(h, dn, chunked=True) for _ in range(3))
        out[key] = max(big, small)
        out[key + "_256mb"] = big
        out[key + "_chunked"] = small
    out["chunk_bytes"] = chunk
    return out


def gemm_kernel_timing(torch, capi, a, reps=20):
    """Average device time per launch of the step's three tcgen05 GEMM shapes, each exactly as
    the executor's bf16 training runs it (forward y = relu(xW + b) also writing the ReLU bit
    mask, dX = (dz W^T) . [x > 0] gated by that mask, dW with its chosen variant: SGD fused
    into the epilogue when one split fills the SMs, else split-K fp32 partials), launched back
    to back on the current stream between two CUDA events, with operands of the step's exact
    shape."""
    rows, d = a.rows, a.d
    x = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
    dz = torch.randn(rows, d, device="cuda").to(torch.bfloat16) * 1e-3
    W = torch.randn(d, d, device="cuda").to(torch.bfloat16)
    W32 = torch.randn(d, d, device="cuda")
    import ctypes
    dw_cta, dw_bn = ctypes.c_int32(), ctypes.c_int32()
    dw_splits = int(capi.LIB.sp_debug_dw_choice(d, rows, 1, ctypes.byref(dw_cta), ctypes.byref(dw_bn)))
    parts = torch.empty(max(dw_splits, 1) * d * d, device="cuda") if dw_splits > 1 else W32
    bias = torch.randn(d, device="cuda")
    out = torch.empty(rows, d, device="cuda", dtype=torch.bfloat16)
    # the executor's bf16 training gates dX with the ReLU bit mask its forward epilogue wrote
    mask = torch.zeros(rows * d // 32, device="cuda", dtype=torch.int32)
    st = torch.cuda.current_stream().cuda_stream
    L = capi.LIB
    shapes = {
        "fwd": (lambda: L.sp_debug_gemm_bf16_masked_async(
            rows, d, d, x.data_ptr(), d, 0, W.data_ptr(), d, 1, 0, out.data_ptr(), d,
            bias.data_ptr(), 1, None, 0, 1, 0, 0, st, mask.data_ptr(), None), a.layers),
        "dx": (lambda: L.sp_debug_gemm_bf16_masked_async(
            rows, d, d, dz.data_ptr(), d, 0, W.data_ptr(), d, 0, 2, out.data_ptr(), d, None, 1,
            x.data_ptr(), d, 1, 0, 0, st, None, mask.data_ptr()), a.layers - 1),
        "dw": (lambda: L.sp_debug_gemm_bf16_async(d, d, rows, x.data_ptr(), d, 1,
                                                  dz.data_ptr(), d, 1, 4 if dw_splits == 1 else 3,
                                                  parts.data_ptr(), d, None, 0, None, 0,
                                                  dw_splits, dw_bn.value, dw_cta.value, st), a.layers),
    }
    res = {}
    for name, (fn, per_step) in shapes.items():
        for _ in range(3):
            assert fn() == 0
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        fl = 2.0 * rows * d * d
        res[name] = {"ms": ms, "flops": fl, "tflops": fl / ms / 1e9, "per_step": per_step}
    return res


def ring_roofline(L, S, lb, opt, fl_f, fl_b, link, pk, ckpt=False, fl_b_first=None, lb_fwd=None, lb_hit=0.0):
    """Ring roofline: a model of the step's lower time bound for a k-window ring of S slots,
    from per-layer FLOPs at the sustained tensor peak and host-link bytes at the measured
    pinned rates.

    Bytes: S slots carry at most S layers across each direction reversal (end of forward, end
    of step), so the forward loads >= L - S layers and the backward >= L - S; every trained
    layer writes its fp32 image (lb bytes) back. AdamW adds the moments m, v (opt bytes) of
    every layer both ways. Up to min(S, L - S) of the write-backs (the layers still resident at
    the end) can run in the next forward, whose D2H engine is otherwise idle (no deferral with
    activation offload).
      forward  = sum over layers of max(FLOP, load / H2D rate), and at least the forward's
                 link bytes (loads + deferred write-backs) at the duplex rate;
      backward = max(sum over layers of max(FLOP, load / duplex rate),
                     its write-backs / D2H rate, its loads + write-backs / (2 x duplex rate)).
    Per-layer serialisation is applied to the loads (a layer computes after its load) but not
    to the write-backs, which overlap later layers' loads. fl_f / fl_b: one layer's forward /
    backward FLOPs (fl_b_first: the bottom layer's, which needs no input gradient). A split
    master (named-shape layers) loads only lb_fwd bytes per forward layer (its bf16 wire prefix)
    and lb_hit bytes for a backward layer still resident (the low halves the update needs)."""
    lb_fwd = lb if lb_fwd is None else lb_fwd
    S = min(S, L)
    peak = pk["bf16_tflops_sustained"] * 1e12
    h2d, d2h, dup = link["h2d_gbs"] * 1e9, link["d2h_gbs"] * 1e9, link["duplex_gbs_per_dir"] * 1e9
    tf, tb = fl_f / peak, fl_b / peak
    tb0 = (fl_b_first if fl_b_first is not None else fl_b) / peak
    deferred = 0 if ckpt else min(S, L - S)
    out_layer = lb + opt
    fwd = (L - S) * max(tf, lb_fwd / h2d) + S * tf
    fwd = max(fwd, ((L - S) * lb_fwd + deferred * out_layer) / (2 * dup), deferred * out_layer / d2h)
    per_layer, loads = 0.0, 0.0
    for pos in range(L):
        fl = tb0 if pos == L - 1 else tb
        load = (lb if pos >= S else lb_hit) + opt
        loads += load
        per_layer += max(fl, load / dup) if load else fl
    outs = (L - deferred) * out_layer
    bwd = max(per_layer, outs / d2h, (loads + outs) / (2 * dup))
    return fwd + bwd


def layer_roofline(a, link, pk, rows_per_gpu, slots, shards=1, ckpt=False):
    """ring_roofline for the dense stand-in (square reference blocks of width a.d)."""
    d = a.d
    lb = (d * d + d) * 4 / shards
    opt = 2 * lb if a.optimizer == "adamw" else 0.0
    fl_f = 2.0 * rows_per_gpu * d * d
    return ring_roofline(a.layers, slots, lb, opt, fl_f, 2 * fl_f, link, pk, ckpt, fl_b_first=fl_f)


def cpu_baseline_ref(a, threads, rows_per_thread=2, layers_sample=6, d=None, layers_full=None):
    """The reference's reference_train_step (oracle/_ref = the reference compiled from its own
    sources) on host cores: `threads` concurrent single-threaded replicas, each training a
    layers_sample-layer slice of d-wide square blocks on rows_per_thread rows. Returns the
    measured seconds and the samples/s of the full model (layers_full square blocks), scaled
    linearly in layers (every block costs the same)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Reference
    ref = Reference()
    d = d or a.d
    layers_full = layers_full or a.layers
    W, b, _ = ref.build_model(7, layers_sample, d)
    xs = [ref.make_input(7, 100 + t, rows_per_thread, d) for t in range(threads)]
    ts = [ref.make_input(7, 200 + t, rows_per_thread, d) for t in range(threads)]
    out = [None] * threads

    def work(t):
        out[t] = ref.train_step(W, b, xs[t], ts[t], a.lr)

    t0 = time.perf_counter()
    th = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    dt = time.perf_counter() - t0
    full = dt * layers_full / layers_sample
    return threads * rows_per_thread / full, dt


REF_ROWS = 16  # rows per host thread per reference-arm step (~1 s of CPU work per step)


def reference_equivalent(a):
    """The reference can only run its square dense block (model.hpp:14-26). The CPU arm of a
    named-shape workload runs reference_train_step on square d-wide blocks carrying the same
    linear-layer FLOPs per token: round(params per layer / d^2) blocks per transformer layer."""
    if a.model == "dense":
        return a.d, a.layers, 1
    from paper_2410_08791_b200 import blocks as B
    spec = B.NAMED_SHAPES[a.model][0]
    lay = B.block_layout(spec)
    per = max(1, round(sum(t.rows * t.cols for t in lay.tensors.values() if t.matrix) / (spec.d * spec.d)))
    return spec.d, a.layers * per, per


def run_reference(a, rank, world):
    if rank != 0:
        return
    threads = max(1, min(os.cpu_count() or 1, 64))
    d, layers_full, per = reference_equivalent(a)
    rates, times = [], []
    for i in range(a.warmup + a.steps):
        v, dt = cpu_baseline_ref(a, threads, rows_per_thread=REF_ROWS, d=d, layers_full=layers_full)
        if i >= a.warmup:
            rates.append(v)
            times.append(dt)
    value = statistics.mean(rates)
    sample = (f"{threads} concurrent reference_train_step replicas x {REF_ROWS} rows x 6 square d={d} "
              f"blocks of the {layers_full}-block FLOP-equivalent model ({per} per layer x {a.layers} layers); "
              f"value scaled x{layers_full / 6:g} in blocks")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": 1e3 * statistics.mean(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_of(a, world),
            "extrapolation": {"measured": "each step trains 6 square blocks on every host thread; "
                                          "ms_per_step is that measured time",
                              "blocks_run": 6, "blocks_full_model": layers_full,
                              "rows_run_per_step": REF_ROWS * threads, "value_scale": layers_full / 6},
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_of(a, world):
    if a.model == "dense":
        return {"workload": f"square-block stand-in: {a.layers} x d={a.d} dense ReLU blocks "
                            f"(reference LayerBlock), bf16 train step (fwd+MSE+bwd+{a.optimizer.upper()})",
                "model": "dense", "layers": a.layers, "d": a.d, "rows_per_gpu": a.rows,
                "global_batch": a.rows * world,
                "strategy": a.strategy, "k": a.k, "k_prime": a.kp, "transfer_mode": a.mode,
                "weights": "pinned host DRAM (fp32 master), streamed per step",
                "host_master": ("one per rank" if world == 1 or a.private_host_copies
                                else "one per node, shared by all ranks (sp_share_host_master)"),
                "optimizer": a.optimizer if a.optimizer == "sgd" else
                "adamw (fp32 m, v in pinned host DRAM, streamed per step)",
                "parallelism": f"dp{world}", "l2": "working set (weights+activations) >> 126 MB L2"}
    from paper_2410_08791_b200 import blocks as B
    spec, _ = B.NAMED_SHAPES[a.model]
    if a.seq_len:
        spec = spec.with_seq(a.seq_len)
    lay = B.block_layout(spec)
    rows = a.seqs * spec.seq_len
    return {"workload": f"{spec.name}-shape stack: {a.layers} transformer layers (d {spec.d}, ff {spec.ff}, "
                        f"{spec.n_heads} heads / {spec.n_kv_heads} kv of {spec.head_dim}, "
                        f"{'causal' if spec.causal else 'bidirectional'} attention), {lay.n_params / 1e6:.2f}M "
                        f"params per layer; bf16 train step (fwd + MSE + bwd + {a.optimizer.upper()})"
                        + (", activation offload" if a.ckpt else ""),
            "model": a.model, "layers": a.layers, "d": spec.d, "ff": spec.ff, "heads": spec.n_heads,
            "kv_heads": spec.n_kv_heads, "seq_len": spec.seq_len, "seqs_per_gpu": a.seqs,
            "rows_per_gpu": rows, "global_batch": rows * world, "sample": "one token (row)",
            "params_per_layer": lay.n_params,
            "strategy": a.strategy, "k": a.k, "k_prime": a.kp, "transfer_mode": a.mode,
            "activation_offload": a.ckpt,
            "weights": "pinned host DRAM (fp32 master), streamed per step",
            "host_master": ("one per rank" if world == 1 or a.private_host_copies
                            else "one per node, shared by all ranks (sp_share_host_master)"),
            "optimizer": a.optimizer if a.optimizer == "sgd" else
            "adamw (fp32 m, v in pinned host DRAM, streamed per step)",
            "parallelism": f"dp{world}", "l2": "working set (weights+activations) >> 126 MB L2"}


def timed_steps(torch, dist, world, steps, fn, collect=None):
    """Device time of `steps` calls of fn between a barrier + synchronize on both sides (CUDA
    events on the current stream, which the executor's streams join every call), max over ranks."""
    from paper_2410_08791_b200 import dp
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = []
    for _ in range(steps):
        out.append(fn())
        if collect is not None:
            collect()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        dist.barrier()
        ms = dp.max_over_ranks(dist, torch, ms)
    return ms, out


def run_block(a, rank, world, local, torch, dist, sp, pk, pk_src, strategy):
    """The named-shape workload (default: C2, GPT-2 XL layers, bf16 train step)."""
    from paper_2410_08791_b200 import blocks as B
    from paper_2410_08791_b200 import dp
    spec, _ = B.NAMED_SHAPES[a.model]
    if a.seq_len:
        spec = spec.with_seq(a.seq_len)
    lay = B.block_layout(spec)
    rows = a.seqs * spec.seq_len
    model = B.build_block_model(spec, 7, a.layers)
    host_copies_note = []

    def make_executor(strat, opt=a.optimizer, ckpt=a.ckpt):
        e = B.BlockExecutor(a.layers, spec, strat, checkpointing=ckpt, device=local, trace=0)
        e.register_model(model)
        if opt == "adamw":
            e.set_optimizer(sp.OPT_ADAMW, 0.9, 0.999, 1e-8, 0.01)
        if world > 1 and not a.private_host_copies:
            tag = f"/sp_bench_{os.environ.get('MASTER_PORT', '0')}_{opt}_{int(ckpt)}_{strat.kind}"
            err = dp.share_host_master(e, dist, local, tag)
            if err:
                host_copies_note.append(f"rank {rank}: private host copy ({err})")
        if world > 1:
            dp.init_executor_dp(e, dist, rank, world)
        return e

    x = sp.make_input(7, 2 * rank, rows, spec.d)
    t = sp.make_input(7, 2 * rank + 1, rows, spec.d)
    x_dev, t_dev = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
    hx, ht = sp.HostBuffer(x.shape), sp.HostBuffer(t.shape)
    hx.array[...] = x
    ht.array[...] = t
    link = measure_link(torch, chunk=min(lay.n_floats * 4, 128 << 20))
    shards = world if world > 1 else 1
    lb = lay.n_floats * 4 / shards
    fl_f = rows * (lay.linear_flops_per_token() + lay.attn_flops_per_token())
    fl_b = rows * (2 * lay.linear_flops_per_token() + 3.5 * lay.attn_flops_per_token())
    # one GPU / all-reduce data parallel: the split master (forward streams the bf16 wire prefix,
    # a resident backward layer loads its low halves); sharded: the fp32 image in 1/world shards
    split = shards == 1
    mat = sum(t.rows * t.cols for t in lay.tensors.values() if t.matrix)
    lb_fwd = lay.wire_bytes if split else lb
    lb_hit = 2.0 * mat if split else 0.0

    def roof(n_slots, opt, ckpt):
        return ring_roofline(a.layers, n_slots, lb, 2 * lb if opt == "adamw" else 0.0, fl_f, fl_b, link, pk, ckpt,
                             lb_fwd=lb_fwd, lb_hit=lb_hit)

    ex = make_executor(strategy)
    dev = lambda e: (lambda: e.train_step_ptr(x_dev.data_ptr(), t_dev.data_ptr(), rows, a.lr, device=True))  # noqa: E731
    step_dev = dev(ex)
    for _ in range(a.warmup):
        step_dev()
    stats = []
    with Clocks(local) as clk:
        ms, losses = timed_steps(torch, dist, world, a.steps, step_dev, lambda: stats.append(ex.stats()))
    step_e2e = lambda: ex.train_step_ptr(hx.ptr, ht.ptr, rows, a.lr, device=False)  # noqa: E731
    step_e2e()
    ms_e2e, _ = timed_steps(torch, dist, world, a.steps, step_e2e)
    last = stats[-1]
    # One extra step with per-op and per-GEMM CUDA events (not timed): the GEMMs inside the
    # step, the stall / compute split.
    ex.set_trace(2)
    step_dev()
    traced = ex.stats()
    ex.set_trace(0)
    ex.close()
    step_s = ms * 1e-3 / a.steps
    roof_s = roof(last["n_slots"], a.optimizer, a.ckpt)
    variants = {}
    # The same step under other settings, timed the same way in the same run: AdamW (north_star:
    # optimizer state in pinned host DRAM), activation offload (the reference's checkpointing),
    # and Standard (every layer resident: the full-residency HBM the window is compared with).
    specs = [] if a.no_variants else [("adamw", strategy, "adamw", a.ckpt), ("offload", strategy, a.optimizer, True),
                                       ("standard", sp.StrategyConfig(sp.STANDARD), a.optimizer, False)]
    for vname, vstrat, vopt, vckpt in specs:
        if vname == "offload" and a.ckpt:
            continue
        ev = make_executor(vstrat, vopt, vckpt)
        fn = dev(ev)
        for _ in range(a.warmup):
            fn()
        vsteps = max(2, a.steps // 2)
        vms, _ = timed_steps(torch, dist, world, vsteps, fn)
        st = ev.stats()
        vroof = roof(st["n_slots"], vopt, vckpt)
        variants[vname] = {"value": world * rows * vsteps / (vms * 1e-3), "unit": "samples/s",
                           "ms_per_step": vms / vsteps, "ring_roofline_ms": vroof * 1e3,
                           "frac_of_ring_roofline": vroof / (vms * 1e-3 / vsteps),
                           "h2d_gb_per_step": st["h2d_bytes"] / 1e9, "d2h_gb_per_step": st["d2h_bytes"] / 1e9,
                           "hbm_reserved_gb": st["hbm_reserved_bytes"] / 1e9,
                           "ledger_peak_gb": st["peak_bytes"] / 1e9, "n_slots": st["n_slots"],
                           "optimizer": vopt, "activation_offload": vckpt,
                           "strategy": ["standard", "cpu_only", "naive", "superpipeline"][vstrat.kind]}
        ev.close()

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        d, layers_full, per = reference_equivalent(a)
        v, dt = cpu_baseline_ref(a, 1, rows_per_thread=64, layers_sample=6, d=d, layers_full=layers_full)
        cpu = {"value": v, "unit": "samples/s", "cores": 1, "kind": "reference",
               "sample": f"reference_train_step (oracle/_ref), 64 rows x 6 square d={d} blocks, {dt:.1f}s; "
                         f"the model as {layers_full} FLOP-equivalent square blocks ({per} per layer), "
                         f"scaled x{layers_full / 6:g} in blocks"}
    gemm_ms, gemm_fl = traced["gemm_ms"], traced["gemm_flops"]
    achieved = gemm_fl / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else 0.0
    peak_tf = pk["bf16_tflops_sustained"]
    traffic, traffic_src = None, None
    tr_path = os.path.join(ROOT, "profiles", "block_gemm_traffic.json")
    if os.path.exists(tr_path):  # per-launch DRAM bytes of the step's GEMMs, one ncu --set full capture
        try:
            tr = json.load(open(tr_path))
            traffic = tr["bytes_per_launch"]
            traffic_src = {k: tr[k] for k in ("algorithmic_bytes_per_launch", "launches_captured", "source")}
        except Exception:
            traffic = None
    value = world * rows * a.steps / (ms * 1e-3)
    e2e = world * rows * a.steps / (ms_e2e * 1e-3)
    std = variants.get("standard", {}).get("hbm_reserved_gb")
    off = variants.get("offload", {}).get("hbm_reserved_gb") if not a.ckpt else last["hbm_reserved_bytes"] / 1e9
    line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (sp_build_block / make_input seed 7)", "config": config_of(a, world),
            "sequences_per_sec": value / spec.seq_len,
            "peak_hbm_gb": {"ledger": last["peak_bytes"] / 1e9,
                            "ledger_weights": last["peak_weight_bytes"] / 1e9,
                            "measured_reserved": last["hbm_reserved_bytes"] / 1e9,
                            "standard_measured_reserved": std,
                            "offload_measured_reserved": off,
                            "reduction_vs_standard": (1 - last["hbm_reserved_bytes"] / 1e9 / std) if std else None,
                            "offload_reduction_vs_standard": (1 - off / std) if (std and off) else None,
                            "full_residency_weights": a.layers * lay.n_floats * 4 / 1e9},
            "north_star": {"layer_roofline_ms": roof_s * 1e3, "measured_ms": step_s * 1e3,
                           "frac_of_layer_roofline": roof_s / step_s, "link": link,
                           "per_layer": {"fwd_flops": fl_f, "bwd_flops": fl_b, "image_bytes": lb,
                                         "fwd_wire_bytes": lb_fwd, "bwd_resident_load_bytes": lb_hit,
                                         "t_fwd_compute_ms": fl_f / (peak_tf * 1e12) * 1e3,
                                         "t_link_ms": lb / (link["h2d_gbs"] * 1e9) * 1e3},
                           "traced_step": {k: traced[k] for k in (
                               "makespan_ms", "compute_ms", "stall_ms", "h2d_bytes", "d2h_bytes", "n_slots",
                               "graph_replays", "gemm_launches", "attn_launches", "attn_flops")},
                           "loss": losses[-1]},
            "roofline": {"bound": "tensor", "kernel": "tcgen05 bf16 GEMMs of the step (4 forward, 8 backward per layer)",
                         "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": f"{pk_src} bf16_tflops_sustained",
                         "gemm_flops_per_step": gemm_fl, "gemm_ms_per_step": gemm_ms,
                         "gemm_launches_per_step": traced["gemm_launches"],
                         "gemm_share_of_step": gemm_ms * 1e-3 / step_s,
                         "method": "CUDA events around every GEMM launch inside one traced step (trace=2) on "
                                   "the compute stream; algorithmic 2MNK FLOPs / summed event time; "
                                   "sustained peak because the kernels run inside a long step"},
            "variants": variants,
            "host_copies_note": host_copies_note or None,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "samples/s",
                    "h2d_bytes_per_step": 2 * rows * spec.d * 4, "d2h_bytes_per_step": 4},
            "gpu_launches": int(sum(s["kernels_launched"] for s in stats)),
            "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    for spec_ in [s for s in a.sweep.split(",") if s]:
        if spec_ == "standard":
            strat, k, kp = sp.StrategyConfig(sp.STANDARD), a.layers, 0
        else:
            k, kp = (int(v) for v in spec_.split(":"))
            strat = (sp.StrategyConfig(sp.NAIVE, k) if kp == 0
                     else sp.StrategyConfig(sp.SUPERPIPELINE, k, kp, sp.BATCH if a.mode == "batch" else sp.SEQUENTIAL))
        e = make_executor(strat)
        fn = dev(e)
        for _ in range(a.warmup):
            fn()
        sms, _ = timed_steps(torch, dist, world, a.steps, fn)
        st = e.stats()
        if rank == 0:
            print(json.dumps({
                "sweep": spec_, "strategy": ["standard", "cpu_only", "naive", "superpipeline"][strat.kind],
                "k": k, "k_prime": kp, "value": world * rows * a.steps / (sms * 1e-3),
                "unit": "samples/s", "ms_per_step": sms / a.steps, "n_slots": st["n_slots"],
                "peak_hbm_gb": {"ledger_weights": st["peak_weight_bytes"] / 1e9, "ledger": st["peak_bytes"] / 1e9,
                                "measured_reserved": st["hbm_reserved_bytes"] / 1e9},
                "h2d_gb_per_step": st["h2d_bytes"] / 1e9, "d2h_gb_per_step": st["d2h_bytes"] / 1e9,
                "layer_roofline_ms": roof(st["n_slots"], a.optimizer, a.ckpt) * 1e3}), flush=True)
        e.close()


def run_block_infer(a, rank, world, local, torch, dist, sp, pk, pk_src, strategy):
    """Named-shape inference (Llama-3-8B layers, 32 x 2048 tokens per GPU, k=4):
    every rank runs its own ring on its own batch from the node's one pinned master - replicas,
    no collective. Weights stream as the bf16 wire image (2 B per matrix parameter)."""
    import ctypes
    from paper_2410_08791_b200 import _capi
    from paper_2410_08791_b200 import blocks as B
    from paper_2410_08791_b200 import dp
    spec, _ = B.NAMED_SHAPES[a.model]
    if a.seq_len:
        spec = spec.with_seq(a.seq_len)
    lay = B.block_layout(spec)
    rows = a.seqs * spec.seq_len
    # inference keeps only the bf16 wire image on the host (SP_BLOCK_INFER_ONLY): a 70B-shape
    # model's fp32 master (274 GB) would not fit a 196 GB host
    ex = B.BlockExecutor(a.layers, spec, strategy, device=local, trace=0,
                         capacity_bytes=int(a.capacity_gb * 1e9), infer_only=True)
    desc = spec.desc()
    distinct = a.distinct_layers or a.layers
    images = []
    for i in range(min(distinct, a.layers)):  # layer by layer: no second full host copy of the model
        params = np.empty(lay.n_floats, np.float32)
        _capi.check(_capi.LIB.sp_build_block(ctypes.byref(desc), 7, i, params.ctypes.data))
        images.append(params)
        if distinct >= a.layers:
            ex.register_block(i, params)
            images = []
    if images:
        for i in range(a.layers):
            ex.register_block(i, images[i % len(images)])
    note = None
    if world > 1 and not a.private_host_copies:
        note = dp.share_host_master(ex, dist, local, f"/sp_bench_infer_{os.environ.get('MASTER_PORT', '0')}")
    x = sp.make_input(7, rank, rows, spec.d)
    x_dev = torch.from_numpy(x).cuda()
    y_dev = torch.empty_like(x_dev)
    hx, hy = sp.HostBuffer(x.shape), sp.HostBuffer(x.shape)
    hx.array[...] = x
    link = measure_link(torch, chunk=min(lay.wire_bytes, 128 << 20))
    step = lambda: ex.forward_ptr(x_dev.data_ptr(), rows, 1, y_dev.data_ptr(), device=True)  # noqa: E731
    for _ in range(a.warmup):
        step()
    stats = []
    with Clocks(local) as clk:
        ms, _ = timed_steps(torch, dist, world, a.steps, step, lambda: stats.append(ex.stats()))
    step_e2e = lambda: ex.forward_ptr(hx.ptr, rows, 1, hy.ptr, device=False)  # noqa: E731
    step_e2e()
    ms_e2e, _ = timed_steps(torch, dist, world, a.steps, step_e2e)
    last = stats[-1]
    ex.set_trace(2)
    step()
    traced = ex.stats()
    ex.set_trace(0)
    peak = pk["bf16_tflops_sustained"] * 1e12
    fl = rows * (lay.linear_flops_per_token() + lay.attn_flops_per_token())
    per_layer = max(fl / peak, lay.wire_bytes / (link["h2d_gbs"] * 1e9))
    loads = int(round(traced["h2d_bytes"] / lay.wire_bytes))  # layers actually streamed per call
    # north_star's per-layer roofline: a streamed layer costs max(FLOPs at peak, wire bytes over
    # the link), a layer still resident from the previous call its FLOPs alone
    roof_s = loads * per_layer + (a.layers - loads) * fl / peak
    step_s = ms * 1e-3 / a.steps
    gemm_ms, gemm_fl = traced["gemm_ms"], traced["gemm_flops"]
    achieved = gemm_fl / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else 0.0
    value = world * rows * a.steps / (ms * 1e-3)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline_infer(a, spec, lay)
    line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (sp_build_block / make_input seed 7)",
            "config": dict(config_of(a, world), workload=f"{spec.name}-shape stack: {a.layers} transformer "
                           f"layers, bf16 inference (run_inference), {a.seqs} x {spec.seq_len} tokens per GPU, "
                           f"{'replicas' if world > 1 else 'one ring'}", mode="inference",
                           parallelism=f"replicas x{world}" if world > 1 else "dp1",
                           capacity_gb=a.capacity_gb or None,
                           distinct_layer_images=min(a.distinct_layers or a.layers, a.layers)),
            "sequences_per_sec": value / spec.seq_len,
            "peak_hbm_gb": {"ledger": last["peak_bytes"] / 1e9, "ledger_weights": last["peak_weight_bytes"] / 1e9,
                            "measured_reserved": last["hbm_reserved_bytes"] / 1e9,
                            "full_residency_weights_bf16": a.layers * lay.wire_bytes / 1e9},
            "north_star": {"layer_roofline_ms": roof_s * 1e3, "measured_ms": step_s * 1e3,
                           "frac_of_layer_roofline": roof_s / step_s, "link": link,
                           "per_layer": {"flops": fl, "wire_bytes": lay.wire_bytes,
                                         "t_compute_ms": fl / peak * 1e3,
                                         "t_link_ms": lay.wire_bytes / (link["h2d_gbs"] * 1e9) * 1e3,
                                         "bound_ms": per_layer * 1e3, "layers_loaded_per_call": loads},
                           "traced_step": {k: traced[k] for k in ("makespan_ms", "compute_ms", "stall_ms", "h2d_bytes",
                                                                   "n_slots", "gemm_launches", "attn_launches",
                                                                   "attn_flops")}},
            "roofline": {"bound": "tensor", "kernel": "tcgen05 bf16 GEMMs of the step (4 per layer)",
                         "achieved": achieved, "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s",
                         "frac": achieved / pk["bf16_tflops_sustained"], "traffic": None,
                         "peak_source": f"{pk_src} bf16_tflops_sustained", "gemm_flops_per_step": gemm_fl,
                         "gemm_ms_per_step": gemm_ms, "gemm_share_of_step": gemm_ms * 1e-3 / step_s,
                         "method": "CUDA events around every GEMM inside one traced call (trace=2)"},
            "host_copies_note": note, "cpu_baseline": cpu,
            "e2e": {"value": world * rows * a.steps / (ms_e2e * 1e-3), "unit": "samples/s",
                    "h2d_bytes_per_step": rows * spec.d * 4, "d2h_bytes_per_step": rows * spec.d * 4},
            "gpu_launches": int(sum(s_["kernels_launched"] for s_ in stats)), "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ex.close()


def cpu_baseline_infer(a, spec, lay):
    """reference_forward (oracle/_ref) on one core over FLOP-equivalent square blocks: one
    d-wide block on 16 rows, scaled to the model's linear FLOPs and the step's rows."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import Reference
    ref = Reference()
    W, b, _ = ref.build_model(7, 1, spec.d)
    xs = ref.make_input(7, 3, 16, spec.d)
    t0 = time.perf_counter()
    ref.forward(W, b, xs)
    dt = time.perf_counter() - t0
    per = lay.linear_flops_per_token() / (2.0 * spec.d * spec.d)  # square blocks per layer
    tokens_per_s = 16 / (dt * per * a.layers)
    return {"value": tokens_per_s, "unit": "samples/s", "cores": 1, "kind": "reference",
            "sample": f"reference_forward (oracle/_ref), one square d={spec.d} block on 16 rows, {dt:.2f}s; "
                      f"scaled to {per:.1f} FLOP-equivalent blocks per layer x {a.layers} layers"}


def spawn_ranks(a):
    """`--gpus N` without a torchrun environment: re-launch this command as N ranks (one
    process per GPU, 127.0.0.1 rendezvous) and return their exit code. Only rank 0 prints."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    if os.environ.get("SP_BENCH_DRY_SPAWN"):  # CPU test: show the launch, do not run it
        print(json.dumps({"spawn": cmd}), flush=True)
        return 0
    return subprocess.call(cmd)


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(a))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != a.gpus:
        print(json.dumps({"error": f"--gpus {a.gpus} but WORLD_SIZE={world}"}), flush=True)
        sys.exit(2)
    if a.impl == "reference":
        run_reference(a, rank, world)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    import paper_2410_08791_b200 as sp
    from paper_2410_08791_b200 import _capi

    pk, pk_src = peaks()
    tmode = sp.BATCH if a.mode == "batch" else sp.SEQUENTIAL
    strategy = {"superpipeline": sp.StrategyConfig(sp.SUPERPIPELINE, a.k, a.kp, tmode),
                "standard": sp.StrategyConfig(sp.STANDARD),
                "naive": sp.StrategyConfig(sp.NAIVE, a.k)}[a.strategy]
    if a.model != "dense" and a.infer:
        run_block_infer(a, rank, world, local, torch, dist, sp, pk, pk_src, strategy)
        if world > 1:
            dist.destroy_process_group()
        return
    if a.model != "dense":
        run_block(a, rank, world, local, torch, dist, sp, pk, pk_src, strategy)
        if world > 1:
            dist.destroy_process_group()
        return
    weights = []  # build_model(7, layers, d) — generated once, registered per executor
    for i in range(a.layers):
        Wl = np.empty((a.d, a.d), np.float32)
        bl = np.empty((a.d,), np.float32)
        _capi.LIB.sp_build_layer(7, i, a.d, 0, 0, Wl.ctypes.data, bl.ctypes.data)
        weights.append((Wl, bl))

    def make_executor(strat, opt=a.optimizer, numerics=sp.BF16):
        e = sp.Executor(a.layers, a.d, strat, numerics=numerics, device=local, trace=0)
        for i, (Wl, bl) in enumerate(weights):
            e.register_layer(i, Wl, bl)
        if opt == "adamw":
            e.set_optimizer(sp.OPT_ADAMW, 0.9, 0.999, 1e-8, 0.01)
        if world > 1 and not a.private_host_copies:
            # every rank of the node streams from one shared pinned master
            tag = f"/sp_bench_{os.environ.get('MASTER_PORT', '0')}_{opt}_{numerics}"
            err = dp.share_host_master(e, dist, local, tag)
            if err:
                host_copies_note.append(f"rank {rank}: private host copy ({err})")
        return e

    from paper_2410_08791_b200 import dp
    host_copies_note = []
    ex = make_executor(strategy)
    if world > 1:
        dp.init_executor_dp(ex, dist, rank, world)  # per-layer NCCL all-reduce of dW/db

    x = sp.make_input(7, 2 * rank, a.rows, a.d)
    t = sp.make_input(7, 2 * rank + 1, a.rows, a.d)
    x_dev = torch.from_numpy(x).cuda()
    t_dev = torch.from_numpy(t).cuda()
    hx = sp.HostBuffer(x.shape)
    ht = sp.HostBuffer(t.shape)
    hx.array[...] = x
    ht.array[...] = t
    link = measure_link(torch, chunk=(a.d * a.d + a.d) * 4)
    torch.cuda.synchronize()

    def step_dev():
        return ex.train_step_ptr(x_dev.data_ptr(), t_dev.data_ptr(), a.rows, a.lr, device=True)

    def step_e2e():
        return ex.train_step_ptr(hx.ptr, ht.ptr, a.rows, a.lr, device=False)

    def barrier():
        if world > 1:
            dist.barrier()

    def timed(fn, collect):
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        losses = []
        for _ in range(a.steps):
            losses.append(fn())
            if collect is not None:
                collect.append(ex.stats())
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        barrier()
        if world > 1:
            ms = dp.max_over_ranks(dist, torch, ms)
        return ms, losses

    for _ in range(a.warmup):
        step_dev()
    step_e2e()
    stats = []
    with Clocks(local) as clk:
        ms, losses = timed(step_dev, stats)
    ms_e2e, _ = timed(step_e2e, None)
    last = stats[-1]
    variants = {}
    # The same step with AdamW (north_star: optimizer state in pinned host DRAM, fused update)
    # and in tf32 numerics (fp32 operands on the tensor cores), timed the same way in the same
    # run; the headline stays the reference's SGD in bf16.
    for vname in ([] if a.optimizer != "sgd" or a.no_variants else ["adamw", "tf32"]):
        ev = make_executor(strategy, "adamw" if vname == "adamw" else "sgd",
                           sp.TF32 if vname == "tf32" else sp.BF16)
        if world > 1:
            dp.init_executor_dp(ev, dist, rank, world)
        for _ in range(a.warmup):
            ev.train_step_ptr(x_dev.data_ptr(), t_dev.data_ptr(), a.rows, a.lr, device=True)
        barrier()
        torch.cuda.synchronize()
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        v0.record()
        for _ in range(a.steps):
            ev.train_step_ptr(x_dev.data_ptr(), t_dev.data_ptr(), a.rows, a.lr, device=True)
        v1.record()
        torch.cuda.synchronize()
        vms = v0.elapsed_time(v1)
        if world > 1:
            vms = dp.max_over_ranks(dist, torch, vms)
        va = argparse.Namespace(**dict(vars(a), optimizer="adamw" if vname == "adamw" else "sgd"))
        # tf32's dense tensor rate is half of bf16's (1.1 vs 2.25 PFLOP/s nominal): the
        # measured sustained bf16 peak / 2 is its roofline denominator
        vpk = dict(pk, bf16_tflops_sustained=pk["bf16_tflops_sustained"] / 2) if vname == "tf32" else pk
        vroof = layer_roofline(va, link, vpk, a.rows, ev.stats()["n_slots"], world if world > 1 else 1)
        variants[vname] = {"value": world * a.rows * a.steps / (vms * 1e-3), "unit": "samples/s",
                           "ms_per_step": vms / a.steps, "ring_roofline_ms": vroof * 1e3,
                           "frac_of_ring_roofline": vroof / (vms * 1e-3 / a.steps),
                           "h2d_gb_per_step": ev.stats()["h2d_bytes"] / 1e9,
                           "d2h_gb_per_step": ev.stats()["d2h_bytes"] / 1e9,
                           "numerics": "tf32" if vname == "tf32" else "bf16",
                           "optimizer": "adamw" if vname == "adamw" else "sgd"}
        ev.close()
    # One extra step with the per-op CUDA-event timeline (not timed): stall / compute split.
    ex.set_trace(1)
    step_dev()
    traced = ex.stats()
    ex.set_trace(0)
    gemm = gemm_kernel_timing(torch, _capi, a)
    gemm_fl = sum(g["flops"] * g["per_step"] for g in gemm.values())
    gemm_s = sum(g["ms"] * 1e-3 * g["per_step"] for g in gemm.values())
    achieved = gemm_fl / gemm_s / 1e12
    gemm_n = sum(g["per_step"] for g in gemm.values())
    peak_tf = pk["bf16_tflops_sustained"]
    traffic, traffic_src = None, None
    tr_path = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tr_path):
        try:
            tr = json.load(open(tr_path))
            traffic, traffic_src = tr.get("bytes_per_launch"), tr.get("source")
        except Exception:
            traffic = None
    step_s = ms * 1e-3 / a.steps
    shards = world if world > 1 else 1  # dp.init_executor_dp: sharded streaming for world > 1
    roof_s = layer_roofline(a, link, pk, a.rows, traced["n_slots"], shards)
    value = world * a.rows * a.steps / (ms * 1e-3)
    e2e = world * a.rows * a.steps / (ms_e2e * 1e-3)

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        v, dt = cpu_baseline_ref(a, 1, rows_per_thread=128, layers_sample=6)
        cpu = {"value": v, "unit": "samples/s", "cores": 1, "kind": "reference",
               "sample": f"reference_train_step (oracle/_ref), 128 rows x 6 of {a.layers} layers "
                         f"d={a.d}, {dt:.1f}s, scaled x{a.layers / 6:g} in layers"}

    line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (build_model/make_input seed 7)", "config": config_of(a, world),
            "peak_hbm_gb": {"ledger": last["peak_bytes"] / 1e9,
                            "ledger_weights": last["peak_weight_bytes"] / 1e9,
                            "measured_reserved": last["hbm_reserved_bytes"] / 1e9,
                            "full_residency_weights": a.layers * (a.d * a.d + a.d) * 4 / 1e9},
            "north_star": {"layer_roofline_ms": roof_s * 1e3, "measured_ms": step_s * 1e3,
                           "frac_of_layer_roofline": roof_s / step_s, "link": link,
                           "traced_step": {k: traced[k] for k in (
                               "makespan_ms", "compute_ms", "stall_ms", "per_item_ms",
                               "h2d_bytes", "d2h_bytes", "n_slots", "graph_replays")},
                           "loss": losses[-1]},
            "roofline": {"bound": "tensor", "kernel": "tcgen05 bf16 GEMM (fwd / dX / dW)",
                         "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": f"{pk_src} bf16_tflops_sustained",
                         "per_shape": gemm, "launches_per_step": gemm_n,
                         "gemm_share_of_step": gemm_s / step_s,
                         "method": "CUDA events around 20 back-to-back launches per shape on the "
                                   "launching stream, step-weighted by launches per step"},
            "variants": variants,
            "host_copies_note": host_copies_note or None,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "samples/s",
                    "h2d_bytes_per_step": 2 * a.rows * a.d * 4, "d2h_bytes_per_step": 4},
            "gpu_launches": int(sum(s["kernels_launched"] for s in stats)),
            "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ex.close()

    # Optional window sweep (BASELINE configs[1]: "window sweep k=1..8"): extra lines, each a
    # separately timed run of the same step; k=1 is the reference's Naive(1) (Superpipeline
    # needs 0 < k' < k, strategy.cpp:29-33).
    for spec in [s for s in a.sweep.split(",") if s]:
        if spec == "standard":
            strat, k, kp = sp.StrategyConfig(sp.STANDARD), a.layers, 0
        else:
            k, kp = (int(v) for v in spec.split(":"))
            strat = (sp.StrategyConfig(sp.NAIVE, k) if kp == 0
                     else sp.StrategyConfig(sp.SUPERPIPELINE, k, kp,
                                            sp.BATCH if a.mode == "batch" else sp.SEQUENTIAL))
        e = make_executor(strat)
        if world > 1:
            dp.init_executor_dp(e, dist, rank, world)
        for _ in range(a.warmup):
            e.train_step_ptr(x_dev.data_ptr(), t_dev.data_ptr(), a.rows, a.lr, device=True)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            e.train_step_ptr(x_dev.data_ptr(), t_dev.data_ptr(), a.rows, a.lr, device=True)
        e1.record()
        torch.cuda.synchronize()
        sms = e0.elapsed_time(e1)
        if world > 1:
            sms = dp.max_over_ranks(dist, torch, sms)
        st = e.stats()
        if rank == 0:
            print(json.dumps({
                "sweep": spec, "strategy": ["standard", "cpu_only", "naive", "superpipeline"][strat.kind],
                "k": k, "k_prime": kp, "value": world * a.rows * a.steps / (sms * 1e-3),
                "unit": "samples/s", "ms_per_step": sms / a.steps, "n_slots": st["n_slots"],
                "peak_hbm_gb": {"ledger_weights": st["peak_weight_bytes"] / 1e9,
                                "ledger": st["peak_bytes"] / 1e9,
                                "measured_reserved": st["hbm_reserved_bytes"] / 1e9},
                "h2d_gb_per_step": st["h2d_bytes"] / 1e9, "d2h_gb_per_step": st["d2h_bytes"] / 1e9,
                "layer_roofline_ms": layer_roofline(a, link, pk, a.rows, st["n_slots"], shards) * 1e3}),
                flush=True)
        e.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
