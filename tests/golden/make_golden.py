"""Regenerates tests/golden/golden.json by running the REFERENCE itself (oracle/_ref, built
from /root/reference sources by oracle/Makefile). Run in the build container:

    python tests/golden/make_golden.py

Each entry records the inputs (configs/*.json of the reference, or SURVEY.md Appendix A
cases) and the reference's outputs: digests, losses (float bits) and ledger peaks.
"""
from __future__ import annotations

import json
import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from pyoracle import BATCH, NAIVE, SEQUENTIAL, STANDARD, SUPERPIPELINE, Reference  # noqa: E402

DEFAULT_RATES = (200.0, 100.0, 0.0, 512.0, 5.12)  # configs/default.json arena


def f32bits(v: float) -> str:
    return struct.pack("<f", float(v)).hex()


def main():
    R = Reference()
    cases = []

    # configs/default.json: 8x16, seed 7, 4 items x 1 row, SP(4,2) batch; plus compare.
    W, b, fz = R.build_model(7, 8, 16)
    xs = np.stack([R.make_input(7, i, 1, 16) for i in range(4)])
    for name, kind, k, kp in [("standard", STANDARD, 0, 0), ("naive", NAIVE, 4, 0),
                              ("superpipeline", SUPERPIPELINE, 4, 2)]:
        rc, y, s = R.run_inference(W, b, xs, kind, k, kp, BATCH, 1 << 30, DEFAULT_RATES)
        cases.append(dict(name=f"default.json/{name}", kind="infer", seed=7, n_layers=8, d=16,
                          n_items=4, rows=1, strategy=kind, k=k, k_prime=kp, mode=BATCH,
                          capacity=1 << 30, rc=rc, digest=s.digest.decode(),
                          peak_bytes=s.peak_bytes, peak_weight_bytes=s.peak_weight_bytes,
                          n_transfers_h2d=s.n_transfers_h2d, n_transfers_d2h=s.n_transfers_d2h,
                          y_head=[float(v) for v in y.reshape(-1)[:8]]))

    # configs/oom_train.json: 12x16, seed 11, b=4, capacity 15000, SP(6,3), lr 0.01.
    W, b, fz = R.build_model(11, 12, 16)
    x = R.make_input(11, 0, 4, 16)
    t = R.make_input(11, 1, 4, 16)
    for name, kind, k, kp in [("superpipeline", SUPERPIPELINE, 6, 3), ("standard", STANDARD, 0, 0)]:
        rc, W2, b2, s = R.run_train_step(W, b, x, t, 0.01, kind, k, kp, BATCH, 15000, DEFAULT_RATES)
        cases.append(dict(name=f"oom_train.json/{name}", kind="train", seed=11, n_layers=12,
                          d=16, rows=4, lr=0.01, strategy=kind, k=k, k_prime=kp, mode=BATCH,
                          capacity=15000, rc=rc,
                          digest=s.digest.decode() if rc == 0 else None,
                          loss_bits=f32bits(s.loss) if rc == 0 else None,
                          peak_bytes=s.peak_bytes if rc == 0 else None))

    # 12x768 inference (window-invariant digest).
    W, b, fz = R.build_model(7, 12, 768)
    xs = np.stack([R.make_input(7, i, 1, 768) for i in range(4)])
    for k, kp in [(2, 1), (4, 2), (8, 3), (11, 10)]:
        rc, y, s = R.run_inference(W, b, xs, SUPERPIPELINE, k, kp, BATCH, 1 << 40, DEFAULT_RATES)
        cases.append(dict(name=f"12x768/sp({k},{kp})", kind="infer", seed=7, n_layers=12, d=768,
                          n_items=4, rows=1, strategy=SUPERPIPELINE, k=k, k_prime=kp, mode=BATCH,
                          capacity=1 << 40, rc=rc, digest=s.digest.decode(),
                          peak_weight_bytes=s.peak_weight_bytes))

    # build_model(7, 2, 768) b=8 reference_train_step lr 0.01.
    W, b, fz = R.build_model(7, 2, 768)
    x = R.make_input(7, 0, 8, 768)
    t = R.make_input(7, 1, 8, 768)
    loss, W2, b2 = R.train_step(W, b, x, t, 0.01)
    cases.append(dict(name="2x768/reference_train_step", kind="train_ref", seed=7, n_layers=2,
                      d=768, rows=8, lr=0.01, loss_bits=f32bits(loss)))

    # Hand timeline model (test_engine.cpp:44-90): build_model(1, 4, 3, 0), 1 item x 1 row.
    W, b, fz = R.build_model(1, 4, 3)
    xs = R.make_input(1, 0, 1, 3)[None]
    rc, y, s = R.run_inference(W, b, xs, SUPERPIPELINE, 2, 1, SEQUENTIAL, 1000,
                               (48.0, 24.0, 0.0, 18.0, 1.0))
    cases.append(dict(name="hand_timeline/sp(2,1)seq", kind="infer", seed=1, n_layers=4, d=3,
                      n_items=1, rows=1, strategy=SUPERPIPELINE, k=2, k_prime=1, mode=SEQUENTIAL,
                      capacity=1000, rc=rc, digest=s.digest.decode(),
                      peak_weight_bytes=s.peak_weight_bytes, peak_bytes=s.peak_bytes,
                      n_transfers_h2d=s.n_transfers_h2d))

    out = dict(generator="tests/golden/make_golden.py (reference compiled from /root/reference "
                         "by oracle/Makefile)", cases=cases)
    path = os.path.join(ROOT, "tests", "golden", "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"wrote {len(cases)} cases to {path}")
    # The reference's shipped experiment configs (data), for the experiment-harness tests.
    cfg_dir = os.path.join(ROOT, "tests", "golden", "configs")
    os.makedirs(cfg_dir, exist_ok=True)
    for name in ("default.json", "oom_train.json"):
        with open(os.path.join("/root/reference/proj/configs", name)) as f:
            cfg = json.load(f)
        with open(os.path.join(cfg_dir, name), "w") as f:
            json.dump(cfg, f, indent=2)
            f.write("\n")
    print(f"wrote reference configs to {cfg_dir}")


if __name__ == "__main__":
    main()
