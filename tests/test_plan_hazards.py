"""Static race check of the executor's op DAG (CPU only).

The executor runs the plan on four CUDA streams (h2d, compute, d2h, update) ordered only by
the plan's dependency edges plus program order within a stream. For every device or pinned
host buffer the plan touches, any two accesses from DIFFERENT streams where at least one
writes must be ordered by happens-before in the same direction as plan order — otherwise the
GPU may execute them concurrently (the bug class behind an activation reload that overtook
its own offload). Buffers modelled:
  slot weights W[s]   H2D(w) writes; COMPUTE reads; UPDATE / fused-SGD COMPUTE(bwd) writes;
                      D2H reads
  bwd act ba[s]       H2D(a) writes; COMPUTE(bwd, slot s) reads
  host act store[L]   ACTSAVE(L) writes; H2D(a, layer L) reads
  fwd act ring fa[i]  COMPUTE(fwd L) reads fa[L%3], writes fa[(L+1)%3]; ACTSAVE(L) reads fa[L%3]
  grad workspace g[i] COMPUTE(bwd L, trainable) writes g[L%2]; UPDATE(L) reads g[L%2]
  host master[L]      D2H(L) writes; H2D(w, L) reads
  AdamW moments MV[s] H2D(o) writes; UPDATE reads+writes; D2H reads (optimizer_state plans)
  host moments[L]     D2H(L) writes; H2D(o, L) reads
"""
import itertools

import pytest

import paper_2410_08791_b200 as sp
from test_cpu_boundary import parse_plan

STREAM = {"H2D": "h2d", "COMPUTE": "comp", "LOSS": "comp", "D2H": "d2h", "ACTSAVE": "d2h",
          "UPDATE": "upd", "ALLGATHER": "upd"}


def accesses(ops, ckpt, frozen, opt=False):
    acc = []  # (op index, resource, is_write)
    for i, op in enumerate(ops):
        k = op["kind"]
        if k == "H2D":
            o = op.get("o", [0] * len(op["layers"]))
            for L, s, w, a, m in zip(op["layers"], op["slots"], op["w"], op["a"], o):
                if w:
                    acc.append((i, ("W", s), True))
                    acc.append((i, ("host", L), False))
                if a:
                    acc.append((i, ("ba", s), True))
                    acc.append((i, ("hact", L), False))
                if m:
                    acc.append((i, ("MV", s), True))
                    acc.append((i, ("hostMV", L), False))
        elif k == "COMPUTE":
            L, s, bwd = op["layer"], op["slot"], op["pass"] == 1
            acc.append((i, ("W", s), False))
            if bwd and not frozen[L]:
                acc.append((i, ("W", s), True))  # fused SGD (one GPU)
                acc.append((i, ("g", L % 2), True))
            if ckpt and bwd:
                acc.append((i, ("ba", s), False))
            if ckpt and not bwd:
                acc.append((i, ("fa", L % 3), False))
                acc.append((i, ("fa", (L + 1) % 3), True))
        elif k == "UPDATE":
            acc.append((i, ("g", op["layer"] % 2), False))
            acc.append((i, ("W", op["slot"]), True))
            if opt:
                acc.append((i, ("MV", op["slot"]), True))
        elif k == "ALLGATHER":  # sharded streaming: completes the slot over NVLink
            for s in op["slots"]:
                acc.append((i, ("W", s), True))
        elif k == "D2H":
            for L, s in zip(op["layers"], op["slots"]):
                acc.append((i, ("W", s), False))
                acc.append((i, ("host", L), True))
                if opt:
                    acc.append((i, ("MV", s), False))
                    acc.append((i, ("hostMV", L), True))
        elif k == "ACTSAVE":
            L = op["layer"]
            acc.append((i, ("fa", L % 3), False))
            acc.append((i, ("hact", L), True))
    return acc


def happens_before(ops):
    n = len(ops)
    preds = [set(op.get("deps", [])) for op in ops]
    last = {}
    for i, op in enumerate(ops):
        st = STREAM[op["kind"]]
        if st in last:
            preds[i].add(last[st])
        last[st] = i
    reach = [0] * n  # bitset of ancestors
    for i in range(n):
        m = 0
        for p in preds[i]:
            m |= reach[p] | (1 << p)
        reach[i] = m
    return lambda a, b: bool(reach[b] >> a & 1)


def check(n, strategy, train, ckpt, items=1, frozen=None, sharded=False, opt=False):
    # both dependency modes: the reference policy's triggers, and eager prefetch (an H2D waits
    # only for its slot) - the executor's default, which must be just as race-free
    for eager in (False, True):
        check_one(n, strategy, train, ckpt, items, frozen, sharded, eager, opt)


def check_one(n, strategy, train, ckpt, items, frozen, sharded, eager, opt=False):
    frozen = frozen or [0] * n
    txt = sp.describe_plan(n, 8, strategy, n_items=items, train=train, checkpointing=ckpt,
                           frozen=frozen, sharded=sharded, eager=eager, optimizer_state=opt)
    assert not txt.startswith("ERROR"), txt
    head, ops = parse_plan(txt)
    ck = ckpt and train and strategy.kind != sp.STANDARD
    hb = happens_before(ops)
    by_res = {}
    for i, res, w in accesses(ops, ck, frozen, opt and train):
        by_res.setdefault(res, []).append((i, w))
    for res, lst in by_res.items():
        for (a, wa), (b, wb) in itertools.combinations(sorted(lst), 2):
            if a == b or not (wa or wb):
                continue
            if STREAM[ops[a]["kind"]] == STREAM[ops[b]["kind"]]:
                continue
            assert hb(a, b), (f"unordered {res}: op {a} {ops[a]['kind']} and op {b} "
                              f"{ops[b]['kind']} (n={n} {strategy} train={train} ckpt={ckpt} "
                              f"eager={eager})")


STRATS = [sp.StrategyConfig(sp.STANDARD), sp.StrategyConfig(sp.NAIVE, 1),
          sp.StrategyConfig(sp.NAIVE, 2), sp.StrategyConfig(sp.SUPERPIPELINE, 2, 1),
          sp.StrategyConfig(sp.SUPERPIPELINE, 3, 1), sp.StrategyConfig(sp.SUPERPIPELINE, 4, 2),
          sp.StrategyConfig(sp.SUPERPIPELINE, 4, 3, sp.SEQUENTIAL)]


@pytest.mark.parametrize("n", [2, 3, 5, 8])
@pytest.mark.parametrize("ckpt", [False, True])
def test_training_plan_has_no_cross_stream_races(n, ckpt):
    for s in STRATS:
        if s.k > n:
            continue
        for frozen in ([0] * n, [1] + [0] * (n - 1), [1] * (n // 2) + [0] * (n - n // 2)):
            check(n, s, True, ckpt, frozen=frozen)


@pytest.mark.parametrize("n,items", [(2, 3), (5, 2), (8, 4)])
def test_inference_plan_has_no_cross_stream_races(n, items):
    for s in STRATS:
        if s.k <= n:
            check(n, s, False, False, items=items)
            check(n, s, False, False, items=items, sharded=True)


@pytest.mark.parametrize("n", [2, 5, 8])
@pytest.mark.parametrize("ckpt", [False, True])
def test_sharded_training_plan_has_no_cross_stream_races(n, ckpt):
    for s in STRATS:
        if s.k <= n:
            for frozen in ([0] * n, [1] + [0] * (n - 1)):
                check(n, s, True, ckpt, frozen=frozen, sharded=True)


@pytest.mark.parametrize("n", [2, 3, 5, 8])
@pytest.mark.parametrize("ckpt", [False, True])
def test_adamw_plan_orders_every_moment_transfer(n, ckpt):
    # AdamW: the moments of every trainable layer ride the backward pass through the ring
    # (H2D o=1 -> UPDATE -> D2H), so the MV region of a slot and the host moments are
    # checked exactly like the weights, sharded and not.
    for s in STRATS:
        if s.k > n:
            continue
        for frozen in ([0] * n, [1] + [0] * (n - 1)):
            check(n, s, True, ckpt, frozen=frozen, opt=True)
            check(n, s, True, ckpt, frozen=frozen, sharded=True, opt=True)


def test_adamw_plan_streams_moments_for_each_trainable_layer_once():
    n = 8
    frozen = [1, 0, 0, 1, 0, 0, 0, 0]
    for s in STRATS:
        head, ops = parse_plan(sp.describe_plan(n, 8, s, train=True, frozen=frozen,
                                                optimizer_state=True))
        moved = [L for o in ops if o["kind"] == "H2D" and o["pass"] == 1
                 for L, m in zip(o["layers"], o["o"]) if m]
        assert sorted(moved) == [L for L in range(n) if not frozen[L]], (s, moved)
        assert not any(m for o in ops if o["kind"] == "H2D" and o["pass"] == 0 for m in o["o"])
        # each moment load precedes (happens-before) the update of that layer
        hb = happens_before(ops)
        load = {L: o["index"] for o in ops if o["kind"] == "H2D"
                for L, m in zip(o["layers"], o["o"]) if m}
        for o in ops:
            if o["kind"] == "UPDATE":
                assert hb(load[o["layer"]], o["index"])


def test_sharded_plan_gathers_every_loaded_layer_and_never_reuses_updated_slots():
    head, ops = parse_plan(sp.describe_plan(8, 8, sp.StrategyConfig(sp.SUPERPIPELINE, 4, 2),
                                            train=True, sharded=True))
    h2d = [o for o in ops if o["kind"] == "H2D"]
    ag = [o for o in ops if o["kind"] == "ALLGATHER"]
    assert len(ag) == len(h2d)
    for o in ag:  # each all-gather directly follows (and depends on) its H2D
        assert ops[o["index"] - 1]["kind"] == "H2D" and o["index"] - 1 in o["deps"]
    # every compute depends on the all-gather that last completed its slot (not the raw H2D)
    fill = {}
    for o in ops:
        if o["kind"] == "ALLGATHER":
            for s in o["slots"]:
                fill[s] = o["index"]
        if o["kind"] == "COMPUTE":
            assert fill[o["slot"]] in o["deps"], o
    # after its backward update a slot holds only this rank's fresh shard: the next step must
    # reload it (final slot cache invalid), checked through the executor on GPU


def test_checker_detects_a_missing_edge():
    # Sanity: drop every dependency edge and the checker must complain.
    txt = sp.describe_plan(4, 8, sp.StrategyConfig(sp.SUPERPIPELINE, 2, 1), train=True,
                           checkpointing=True)
    head, ops = parse_plan(txt)
    for op in ops:
        op["deps"] = []
    hb = happens_before(ops)
    bad = 0
    by_res = {}
    for i, res, w in accesses(ops, True, [0] * 4):
        by_res.setdefault(res, []).append((i, w))
    for res, lst in by_res.items():
        for (a, wa), (b, wb) in itertools.combinations(sorted(lst), 2):
            if (wa or wb) and STREAM[ops[a]["kind"]] != STREAM[ops[b]["kind"]] and not hb(a, b):
                bad += 1
    assert bad > 0


def test_eager_prefetch_changes_only_the_trigger_dependencies():
    """Eager prefetch keeps the op sequence, slots and ledger of the reference policy; H2D ops
    only lose the dependency on their trigger compute (so copies can run ahead into free
    slots), and every other op's dependencies are unchanged."""
    for train in (False, True):
        a = parse_plan(sp.describe_plan(12, 8, sp.StrategyConfig(sp.SUPERPIPELINE, 2, 1), train=train))[1]
        b = parse_plan(sp.describe_plan(12, 8, sp.StrategyConfig(sp.SUPERPIPELINE, 2, 1), train=train,
                                        eager=True))[1]
        assert len(a) == len(b)
        relaxed = 0
        for x, y in zip(a, b):
            assert {k: v for k, v in x.items() if k != "deps"} == {k: v for k, v in y.items() if k != "deps"}
            assert set(y["deps"]) <= set(x["deps"])
            if x["kind"] != "H2D":
                assert x["deps"] == y["deps"]
            relaxed += len(set(x["deps"]) - set(y["deps"]))
        assert relaxed > 0
