"""Tuner parity with the reference's grid_search semantics (test_tuner.cpp:53-156,
acceptance C8): grid size, pre-filter, feasibility, tie-break. CPU cases use a deterministic
fake evaluator; the GPU case measures on the device."""
import pytest

import paper_2410_08791_b200 as sp
from paper_2410_08791_b200 import tuner


def fake_evaluator(n_layers, layer_bytes):
    def evaluate(s):
        peak = min(s.k + s.k_prime, n_layers) * layer_bytes + 16 * 4
        return peak, 10.0 / s.k + 1.0 / s.k_prime  # faster with larger windows
    return evaluate


def test_grid_has_28_pairs_for_k_2_to_8():
    model = sp.build_model(7, 8, 16)
    spec = tuner.SweepSpec(2, 8, 1, 7, 1 << 40, tuner.MIN_PER_ITEM_TIME)
    r = tuner.grid_search(model, sp.ArenaConfig(), tuner.SweepWorkload(2, 1), spec,
                          evaluate=fake_evaluator(8, model.layer_bytes()))
    assert len(r.table) == 28  # acceptance.cpp:352 / test_tuner.cpp:59
    assert [(e.k, e.k_prime) for e in r.table][:3] == [(2, 1), (3, 1), (3, 2)]
    assert r.best == (8, 7)


def test_budget_prefilter_and_min_peak_objective():
    model = sp.build_model(7, 8, 16)
    lb = model.layer_bytes()
    spec = tuner.SweepSpec(2, 8, 1, 7, 5 * lb + 64, tuner.MIN_TIME_UNDER_BUDGET)
    r = tuner.grid_search(model, sp.ArenaConfig(), tuner.SweepWorkload(1, 1), spec,
                          evaluate=fake_evaluator(8, lb))
    feas = [(e.k, e.k_prime) for e in r.table if e.feasible]
    assert all(k + kp <= 5 for k, kp in feas) and feas
    assert r.best in feas
    spec.objective = tuner.MIN_PEAK_BYTES
    r = tuner.grid_search(model, sp.ArenaConfig(), tuner.SweepWorkload(1, 1), spec,
                          evaluate=fake_evaluator(8, lb))
    assert r.best == (2, 1)  # smallest window; ties broken by k then k'


def test_tie_break_order():
    a = tuner.SweepEntry(3, 1, True, 100, 1.0)
    b = tuner.SweepEntry(2, 1, True, 100, 1.0)
    c = tuner.SweepEntry(2, 1, True, 90, 1.0)
    assert tuner.better(tuner.MIN_PER_ITEM_TIME, b, a)
    assert tuner.better(tuner.MIN_PER_ITEM_TIME, c, b)


def test_spec_validation():
    with pytest.raises(sp.InvalidArgument):
        tuner.SweepSpec(2, 8, 1, 7, 0).validate()
    with pytest.raises(sp.InvalidArgument):
        tuner.SweepSpec(5, 2, 1, 1, 10).validate()


@pytest.mark.gpu
def test_gpu_grid_search_measures_and_respects_budget():
    model = sp.build_model(7, 12, 256)
    lb = model.layer_bytes()
    spec = tuner.SweepSpec(2, 6, 1, 3, 7 * lb + 512 * 256 * 4, tuner.MIN_TIME_UNDER_BUDGET)
    wl = tuner.SweepWorkload(1, 512)
    r = tuner.grid_search(model, sp.ArenaConfig(), wl, spec,
                          evaluate=tuner.gpu_evaluator(model, wl, repeats=2))
    assert r.best is not None
    for e in r.table:
        if e.feasible:
            assert e.peak_bytes <= spec.budget_bytes and e.per_item_time > 0
    k, kp = r.best
    assert k + kp <= 7
