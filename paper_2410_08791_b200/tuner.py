"""(k, k') grid search with the GPU executor as the evaluator.

Mirrors the reference tuner (tuner.hpp:16-55, tuner.cpp:48-105): the same SweepSpec /
SweepEntry / SweepResult, the same grid order (k ascending, then k'), the same analytic
pre-filter (peak weight residency + one activation buffer > budget => skip), the same
feasibility rule (peak_bytes <= budget) and tie-break (objective, then peak bytes, then k,
then k'). The objective's time is MEASURED on the GPU (median of `repeats` device-timed
calls) instead of the simulator's virtual clock; training workloads are supported too.
"""
from __future__ import annotations

import statistics
from dataclasses import dataclass, field

import numpy as np

from . import engine as E

MIN_PER_ITEM_TIME, MIN_PEAK_BYTES, MIN_TIME_UNDER_BUDGET = range(3)  # tuner.hpp:16


@dataclass
class SweepSpec:
    k_min: int = 2
    k_max: int = 2
    k_prime_min: int = 1
    k_prime_max: int = 1
    budget_bytes: int = 0
    objective: int = MIN_TIME_UNDER_BUDGET

    def validate(self):  # tuner.cpp:14-22
        if self.k_min > self.k_max or self.k_prime_min > self.k_prime_max:
            raise E.InvalidArgument(2, "sweep: empty range")
        if self.k_min < 1 or self.k_prime_min < 1:
            raise E.InvalidArgument(2, "sweep: ranges must be positive")
        if self.budget_bytes == 0:
            raise E.InvalidArgument(2, "sweep: budget_bytes must be > 0")


@dataclass
class SweepWorkload:
    n_items: int = 1
    batch_size: int = 1
    transfer_mode: int = E.BATCH
    train: bool = False
    lr: float = 0.01


@dataclass
class SweepEntry:
    k: int
    k_prime: int
    feasible: bool = False
    peak_bytes: int = 0
    per_item_time: float = 0.0  # seconds of device time


@dataclass
class SweepResult:
    table: list = field(default_factory=list)
    best: tuple | None = None


def better(objective: int, a: SweepEntry, b: SweepEntry) -> bool:
    """tuner.cpp:27-44."""
    if objective == MIN_PEAK_BYTES:
        pa, pb = float(a.peak_bytes), float(b.peak_bytes)
    else:
        pa, pb = a.per_item_time, b.per_item_time
    if pa != pb:
        return pa < pb
    if a.peak_bytes != b.peak_bytes:
        return a.peak_bytes < b.peak_bytes
    if a.k != b.k:
        return a.k < b.k
    return a.k_prime < b.k_prime


def pick_best(table, objective):
    best = None
    for e in table:
        if e.feasible and (best is None or better(objective, e, best)):
            best = e
    return None if best is None else (best.k, best.k_prime)


def gpu_evaluator(model: E.LayeredModel, workload: SweepWorkload, numerics=E.BF16, repeats=3,
                  capacity_bytes=0):
    """Returns evaluate(strategy) -> (peak_bytes, per_item_time_s) measured on the GPU."""
    inputs = np.stack([E.make_input(model.seed, i, workload.batch_size, model.d)
                       for i in range(workload.n_items)])
    target = E.make_input(model.seed, 1002, workload.batch_size, model.d)

    def evaluate(strategy: E.StrategyConfig):
        with E.Executor(model.n_layers, model.d, strategy, numerics=numerics, trace=0,
                        capacity_bytes=capacity_bytes) as ex:
            ex.register_model(model)
            times = []
            for r in range(repeats + 1):
                if workload.train:
                    ex.train_step(inputs[0], target, workload.lr)
                else:
                    ex.forward(inputs)
                if r:  # first call captures the graph
                    times.append(ex.stats()["makespan_ms"] * 1e-3)
            st = ex.stats()
            return st["peak_bytes"], statistics.median(times) / workload.n_items

    return evaluate


def grid_search(model: E.LayeredModel, arena: E.ArenaConfig, workload: SweepWorkload,
                spec: SweepSpec, evaluate=None) -> SweepResult:
    """tuner.cpp:48-105 with a measured objective."""
    spec.validate()
    if workload.n_items < 1 or workload.batch_size < 1:
        raise E.InvalidArgument(2, "sweep: workload counts must be >= 1")
    evaluate = evaluate or gpu_evaluator(model, workload, capacity_bytes=arena.capacity_bytes)
    act_bytes = workload.batch_size * model.d * 4
    result = SweepResult()
    for k in range(spec.k_min, spec.k_max + 1):
        for kp in range(spec.k_prime_min, spec.k_prime_max + 1):
            if kp >= k or k > model.n_layers:
                continue
            s = E.StrategyConfig(E.SUPERPIPELINE, k, kp, workload.transfer_mode)
            entry = SweepEntry(k, kp)
            bound = E.peak_weight_residency(s, model.n_layers, model.layer_bytes()) + act_bytes
            if bound > spec.budget_bytes:
                result.table.append(entry)
                continue
            try:
                entry.peak_bytes, entry.per_item_time = evaluate(s)
                entry.feasible = entry.peak_bytes <= spec.budget_bytes
            except E.OomDeadlockError:
                entry.feasible = False
            result.table.append(entry)
    result.best = pick_best(result.table, spec.objective)
    return result
