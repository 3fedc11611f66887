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
  write-back stage[i] UPDATE(stage=i) writes (copy of its slot); D2H(stage=i) reads it instead
                      of the slot. A deferred D2H moves nothing in its call; the next call's
                      plan starts with that write-back (SP_PLAN_WRITEBACK shows the steady state)
An H2D job is checked as one sub-op per moved layer, in stream order, as the executor runs
it: with eager prefetch each moved layer waits for its own dependencies (md=) right before its
copy (otherwise the job's first copy waits for all of them), and a COMPUTE that depends on the
job waits only for the sub-op that moved its own layer (a per-move completion event); every
other dependent waits for the whole job.
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
            if op.get("stage") is not None:
                acc.append((i, ("stage", op["stage"]), True))
        elif k == "ALLGATHER":  # sharded streaming: completes the slot over NVLink
            for s in op["slots"]:
                acc.append((i, ("W", s), True))
        elif k == "D2H":
            if op.get("deferred"):
                continue  # nothing moves in this call
            for L, s in zip(op["layers"], op["slots"]):
                src = ("stage", op["stage"]) if op.get("stage") is not None else ("W", s)
                acc.append((i, src, False))
                acc.append((i, ("host", L), True))
                if opt:
                    if op.get("stage") is None:
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


def split_moves(ops, eager=True):
    """One sub-op per moved layer of each H2D job (see the module docstring)."""
    last, first, out = {}, {}, []
    by_index = {op["index"]: op for op in ops}

    def dep_of(op, d):
        src = by_index[d]
        if op["kind"] == "COMPUTE" and src["kind"] == "H2D":
            for j, (L, s) in enumerate(zip(src["layers"], src["slots"])):
                if L == op["layer"] and s == op["slot"]:
                    return first[d] + j
        return last[d]

    for op in ops:
        if op["kind"] == "H2D" and len(op["layers"]) > 0:
            first[op["index"]] = len(out)
            for j in range(len(op["layers"])):
                sub = {k: ([v[j]] if k in ("layers", "slots", "w", "a", "o") and isinstance(v, list) else v)
                       for k, v in op.items()}
                if eager and op.get("md") is not None:
                    sub["deps"] = [last[d] for d in (op["md"][j] if j < len(op["md"]) else [])]
                else:
                    sub["deps"] = [last[d] for d in op["deps"]] if j == 0 else []
                sub["index"] = len(out)
                out.append(sub)
        else:
            out.append(dict(op, deps=[dep_of(op, d) for d in op["deps"]], index=len(out)))
        last[op["index"]] = len(out) - 1
    return out


def check(n, strategy, train, ckpt, items=1, frozen=None, sharded=False, opt=False):
    # both dependency modes: the reference policy's triggers, and eager prefetch (an H2D waits
    # only for its slot) - the executor's default, which must be just as race-free; training
    # also with the executor's write-back scheme (staged + deferred, steady state)
    for eager in (False, True):
        for wb in ((False, True) if train else (False,)):
            check_one(n, strategy, train, ckpt, items, frozen, sharded, eager, opt, wb)


def check_one(n, strategy, train, ckpt, items, frozen, sharded, eager, opt=False, wb=False):
    frozen = frozen or [0] * n
    txt = sp.describe_plan(n, 8, strategy, n_items=items, train=train, checkpointing=ckpt,
                           frozen=frozen, sharded=sharded, eager=eager, optimizer_state=opt,
                           writeback=wb)
    assert not txt.startswith("ERROR"), txt
    head, ops = parse_plan(txt)
    ops = split_moves(ops, eager)
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
                              f"eager={eager} writeback={wb} opt={opt})")


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


def _violations(ops, ckpt, frozen, opt=False):
    hb = happens_before(ops)
    by_res, bad = {}, 0
    for i, res, w in accesses(ops, ckpt, frozen, opt):
        by_res.setdefault(res, []).append((i, w))
    for res, lst in by_res.items():
        for (a, wa), (b, wb) in itertools.combinations(sorted(lst), 2):
            if (wa or wb) and a != b and STREAM[ops[a]["kind"]] != STREAM[ops[b]["kind"]] and not hb(a, b):
                bad += 1
    return bad


@pytest.mark.parametrize("opt", [False, True])
def test_writeback_scheme_edges_are_each_necessary(opt):
    """The staged / deferred write-back plan is race-free (above) and each of its new edges is
    load-bearing: dropping the waits on the previous call's write-backs, or on a stage's last
    reader, or one moved layer's own md deps, makes the checker fire."""
    n, s = 16, sp.StrategyConfig(sp.SUPERPIPELINE, 4, 2)  # 10 staged write-backs > 3 stages
    txt = sp.describe_plan(n, 8, s, train=True, eager=True, writeback=True, optimizer_state=opt)
    head, ops = parse_plan(txt)
    pend = {o["index"] for o in ops if o["kind"] == "D2H" and o["pass"] == 0}
    assert pend and any(o.get("deferred") for o in ops) and any(o.get("stage") is not None for o in ops)
    base = split_moves(ops)
    assert _violations(base, False, [0] * n, opt) == 0

    def drop(pred):
        cut = [dict(o) for o in ops]
        for o in cut:
            o["deps"] = [d for d in o["deps"] if not pred(o, d)]
            if o.get("md") is not None:
                o["md"] = [[d for d in md if not pred(o, d)] for md in o["md"]]
        return split_moves(cut)

    assert _violations(drop(lambda o, d: d in pend), False, [0] * n, opt) > 0
    stage_readers = {o["index"] for o in ops if o["kind"] == "D2H" and o.get("stage") is not None}
    assert _violations(drop(lambda o, d: o["kind"] == "UPDATE" and d in stage_readers),
                       False, [0] * n, opt) > 0
    # the per-move split itself: give every move the first move's deps only
    cut = [dict(o) for o in ops]
    for o in cut:
        if o["kind"] == "H2D" and len(o.get("md") or []) > 1:
            o["md"] = [o["md"][0]] + [[] for _ in o["md"][1:]]
    assert _violations(split_moves(cut), False, [0] * n, opt) > 0


def test_writeback_scheme_keeps_policy_ops_and_moves_tail_writebacks():
    """Same backward compute / H2D sequence as the plain plan; the trained layers still
    resident at the end (the ring's last S backward layers) are written back by the next call."""
    n, s = 12, sp.StrategyConfig(sp.SUPERPIPELINE, 4, 2)
    plain = parse_plan(sp.describe_plan(n, 8, s, train=True, eager=True))[1]
    steady = parse_plan(sp.describe_plan(n, 8, s, train=True, eager=True, writeback=True))[1]
    key = lambda o: (o["kind"], o.get("layer"), o.get("layers"), o.get("slots"))  # noqa: E731
    # (the plain plan is a cold first call: compare the backward, which starts from the same
    # ring state either way)
    assert [key(o) for o in plain if o["kind"] in ("COMPUTE", "H2D") and o["pass"] == 1] == \
        [key(o) for o in steady if o["kind"] in ("COMPUTE", "H2D") and o["pass"] == 1]
    pending = [o["layers"][0] for o in steady if o["kind"] == "D2H" and o["pass"] == 0]
    deferred = [o["layers"][0] for o in steady if o.get("deferred")]
    assert sorted(pending) == sorted(deferred) == list(range(6))  # S = k + k' = 6
    assert pending == sorted(pending)  # forward order: the first slot reused is freed first


def _two_calls(n, d, k, kp, cap, act1, act2):
    from paper_2410_08791_b200 import _capi as capi
    import ctypes as C
    cfg = capi.SpConfig(n_layers=n, d=d, strategy=SUPERPIPELINE_, k=k, k_prime=kp,
                        transfer_mode=1, numerics=0, checkpointing=0, device=0, trace=0,
                        capacity_bytes=cap)
    need = capi.LIB.sp_debug_plan_two_calls(C.byref(cfg), act1, act2, None, 0)
    buf = C.create_string_buffer(int(need))
    capi.LIB.sp_debug_plan_two_calls(C.byref(cfg), act1, act2, buf, need)
    return buf.value.decode()


SUPERPIPELINE_ = 3


def test_growing_batch_under_capacity_never_drops_a_deferred_writeback():
    # n=8, SP(4,2), capacity 5600 B, d=16 (1088-B layers). Call 1 at 10 B of
    # activations per layer runs a 5-slot ring and defers the write-backs of the layers still
    # resident; call 2 at 600 B (a larger batch) shrinks the ring below their slots. Every
    # deferred layer must either get its D2H at the start of call 2 or be flushed (completed)
    # before call 2 is planned; before the fix the shrunk plan silently skipped them.
    text = _two_calls(8, 16, 4, 2, 5600, 10, 600)
    lines = text.splitlines()
    deferred = [int(x) for x in lines[0].split()[1:]]
    assert deferred, text
    flushed = []
    body = lines[1:]
    if body and body[0].startswith("FLUSHED"):
        flushed = [int(x) for x in body[0].split()[1:]]
        body = body[1:]
    head, ops = parse_plan("\n".join(body))
    leading = []
    for op in ops:
        if op["kind"] != "D2H":
            break
        leading += op["layers"]
    for L in deferred:
        assert L in flushed or L in leading, (L, text)
    # the scenario really shrinks the ring: the pending write-backs could not all be kept
    assert flushed == deferred


def test_steady_batch_keeps_deferred_writebacks_pending():
    text = _two_calls(8, 16, 4, 2, 0, 100, 100)
    lines = text.splitlines()
    deferred = [int(x) for x in lines[0].split()[1:]]
    assert deferred and not lines[1].startswith("FLUSHED")
    head, ops = parse_plan("\n".join(lines[1:]))
    leading = [L for op in ops[:len(deferred)] if op["kind"] == "D2H" for L in op["layers"]]
    assert sorted(leading) == sorted(deferred)
