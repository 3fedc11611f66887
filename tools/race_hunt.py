"""Repeats small exact-mode training steps and reports any run whose result differs from the
oracle (bitwise). Used to hunt ordering bugs between the executor's streams."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2410_08791_b200 as sp  # noqa: E402
from pyoracle import Oracle  # noqa: E402

orc = Oracle()
cases = [(2033619272433572838, 2, 4, 1, 1), (3234164630432676636, 6, 6, 4, 2), (7, 4, 5, 2, 3)]
strategies = {"standard": sp.StrategyConfig(sp.STANDARD), "naive1": sp.StrategyConfig(sp.NAIVE, 1),
              "naive2": sp.StrategyConfig(sp.NAIVE, 2), "sp21": sp.StrategyConfig(sp.SUPERPIPELINE, 2, 1)}
bad = {}
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for seed, n, d, frozen, b in cases:
    model = sp.build_model(seed, n, d, frozen)
    x, t = sp.make_input(seed, 1001, b, d), sp.make_input(seed, 1002, b, d)
    loss, Wn, bn = orc.train_step(model.W, model.b, x, t, 0.02, frozen=model.frozen)
    for name, s in strategies.items():
        if s.kind == sp.NAIVE and s.k > n:
            continue
        for ckpt in (False, True):
            for r in range(reps):
                rt = sp.run_train_step(model, x, t, s, sp.ArenaConfig(1 << 40), sp.TrainConfig(0.02, ckpt, b))
                ok = np.array_equal(rt.model.W, Wn) and np.array_equal(rt.model.b, bn)
                okl = np.float32(rt.loss) == loss
                if not (ok and okl):
                    key = (seed, n, name, ckpt)
                    bad[key] = bad.get(key, 0) + 1
                    if bad[key] == 1:
                        diffW = [int(np.sum(rt.model.W[l] != Wn[l])) for l in range(n)]
                        diffb = [int(np.sum(rt.model.b[l] != bn[l])) for l in range(n)]
                        print("MISMATCH", key, "loss_ok", bool(okl), "W diffs/layer", diffW, "b diffs", diffb, flush=True)
print("summary", {str(k): v for k, v in bad.items()}, "reps", reps)
