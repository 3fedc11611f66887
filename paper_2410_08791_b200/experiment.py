"""Experiment harness over the GPU executor: the reference's JSON experiment schema and its
run / compare / sweep entry points, as a caller-side data format.

Mirrors experiment.hpp / experiment.cpp of the reference:
  load_config        experiment.cpp:140-216  strict schema (unknown keys rejected at every
                                             level, typed fields, ConfigError on any defect)
  ExperimentConfig.validate                  experiment.cpp:118-138 cross-field invariants
  output_dir         experiment.cpp:218-222  explicit dir, then PIPESIM_OUTPUT_DIR, then "out"
  cmd_run            experiment.cpp:224-243  trace.csv + summary.json, one summary line
  cmd_compare        experiment.cpp:245-291  Standard / CpuOnly / Naive / Superpipeline table
                                             (compare.csv), digest agreement (exit 4)
  cmd_sweep          experiment.cpp:293-325  (k, k') grid -> sweep.csv + "best k=.."
  run_command        main.cpp:160-178        exception -> exit code (2 config, 3 OOM, 1 other)
Differences, all because the executor is real rather than simulated:
  * times are measured device seconds (CUDA events), not virtual seconds;
  * CpuOnly has no GPU path: its compare row reports the reference ledger's peak (0 bytes, no
    weight is ever admitted) and no time ("nan"), and it takes no part in the digest check;
  * the numerics mode (exact fp32 reference order, or bf16 tensor cores) is a call argument,
    not a schema key, so reference configs load unchanged.
There is no command-line front end; callers pass a config path or an ExperimentConfig.
"""
from __future__ import annotations

import json
import math
import os
import sys
from dataclasses import dataclass, field

import numpy as np

from . import engine as E
from . import trace_io, tuner

KIND_NAMES = {"standard": E.STANDARD, "cpu_only": E.CPU_ONLY, "naive": E.NAIVE,
              "superpipeline": E.SUPERPIPELINE}
KIND_OF = {v: k for k, v in KIND_NAMES.items()}
MODE_NAMES = {"batch": E.BATCH, "sequential": E.SEQUENTIAL}
OBJECTIVES = {"min_per_item_time": tuner.MIN_PER_ITEM_TIME, "min_peak_bytes": tuner.MIN_PEAK_BYTES,
              "min_time_under_budget": tuner.MIN_TIME_UNDER_BUDGET}


class ConfigError(ValueError):
    """Invalid, inconsistent, or unknown configuration input (experiment.hpp:17-20): exit 2."""


@dataclass
class ModelSpec:
    seed: int = 1
    n_layers: int = 1
    d: int = 1
    frozen_prefix: int = 0


@dataclass
class WorkloadConfig:
    mode: str = "infer"
    n_items: int = 1
    batch_size: int = 1
    lr: float = 0.01
    checkpointing: bool = False


@dataclass
class OutputConfig:
    dir: str | None = None
    formats: list = field(default_factory=lambda: ["csv", "json"])


@dataclass
class ExperimentConfig:
    model: ModelSpec = field(default_factory=ModelSpec)
    arena: E.ArenaConfig = field(default_factory=E.ArenaConfig)
    workload: WorkloadConfig = field(default_factory=WorkloadConfig)
    strategy: E.StrategyConfig = field(default_factory=E.StrategyConfig)
    output: OutputConfig = field(default_factory=OutputConfig)
    sweep: tuner.SweepSpec | None = None

    def validate(self) -> None:
        m, w = self.model, self.workload
        if m.n_layers < 1:
            raise ConfigError("config: model.n_layers must be >= 1")
        if m.d < 1:
            raise ConfigError("config: model.d must be >= 1")
        if m.frozen_prefix < 0 or m.frozen_prefix > m.n_layers:
            raise ConfigError("config: model.frozen_prefix must be in [0, n_layers]")
        if w.mode not in ("infer", "train"):
            raise ConfigError("config: workload.mode must be 'infer' or 'train'")
        if w.n_items < 1:
            raise ConfigError("config: workload.n_items must be >= 1")
        if w.batch_size < 1:
            raise ConfigError("config: workload.batch_size must be >= 1")
        if not w.lr > 0.0:
            raise ConfigError("config: workload.lr must be > 0")
        for fmt in self.output.formats:
            if fmt not in ("csv", "json"):
                raise ConfigError("config: output.formats entries must be 'csv' or 'json'")
        try:
            self.arena.validate()
            self.strategy.validate(m.n_layers)
            if self.sweep is not None:
                self.sweep.validate()
        except E.InvalidArgument as e:
            raise ConfigError(f"config: {_message(e)}") from e


def _message(e: Exception) -> str:
    text = str(e)
    return text.split("] ", 1)[1] if text.startswith("[sp_status") else text


# ---- strict schema ------------------------------------------------------------------------

def _require_object(j, section):
    if not isinstance(j, dict):
        raise ConfigError(f"config: section '{section}' must be an object")


def _reject_unknown(j, section, allowed):
    for key in j:
        if key not in allowed:
            raise ConfigError(f"config: unknown key '{section}.{key}'")


def _get(j, section, key, kind, fallback):
    """get_field<T> (experiment.cpp:34-42): absent -> fallback; wrong JSON type -> ConfigError.
    Numbers convert like nlohmann's get<T> (a float read as an int truncates); booleans are
    not numbers and numbers are not booleans."""
    if key not in j:
        return fallback
    v = j[key]
    bad = ConfigError(f"config: bad value for '{section}.{key}'")
    if kind in (int, "u64"):
        if isinstance(v, bool) or not isinstance(v, (int, float)) or not math.isfinite(v):
            raise bad
        v = int(v)
        if kind == "u64":
            v &= (1 << 64) - 1  # get<uint64_t> of a negative number wraps
        return v
    if kind is float:
        if isinstance(v, bool) or not isinstance(v, (int, float)):
            raise bad
        return float(v)
    if kind is bool:
        if not isinstance(v, bool):
            raise bad
        return v
    if kind is str:
        if not isinstance(v, str):
            raise bad
        return v
    if kind == "strlist":
        if not isinstance(v, list) or not all(isinstance(x, str) for x in v):
            raise bad
        return list(v)
    raise TypeError(kind)


def parse_config(j) -> ExperimentConfig:
    """The schema of load_config applied to an already-parsed JSON document."""
    _require_object(j, "<root>")
    _reject_unknown(j, "<root>", ("model", "arena", "workload", "strategy", "output", "sweep"))
    cfg = ExperimentConfig()
    if "model" in j:
        m = j["model"]
        _require_object(m, "model")
        _reject_unknown(m, "model", ("seed", "n_layers", "d", "frozen_prefix"))
        cfg.model.seed = _get(m, "model", "seed", "u64", cfg.model.seed)
        cfg.model.n_layers = _get(m, "model", "n_layers", int, cfg.model.n_layers)
        cfg.model.d = _get(m, "model", "d", int, cfg.model.d)
        cfg.model.frozen_prefix = _get(m, "model", "frozen_prefix", int, 0)
    if "arena" in j:
        a = j["arena"]
        _require_object(a, "arena")
        _reject_unknown(a, "arena", ("capacity_bytes", "h2d_bandwidth", "d2h_bandwidth",
                                     "per_call_latency", "device_compute_rate", "host_compute_rate"))
        cfg.arena.capacity_bytes = _get(a, "arena", "capacity_bytes", "u64", cfg.arena.capacity_bytes)
        cfg.arena.h2d_bandwidth = _get(a, "arena", "h2d_bandwidth", float, 1.0)
        cfg.arena.d2h_bandwidth = _get(a, "arena", "d2h_bandwidth", float, 1.0)
        cfg.arena.per_call_latency = _get(a, "arena", "per_call_latency", float, 0.0)
        cfg.arena.device_compute_rate = _get(a, "arena", "device_compute_rate", float, 1.0)
        cfg.arena.host_compute_rate = _get(a, "arena", "host_compute_rate", float, 1.0)
    if "workload" in j:
        w = j["workload"]
        _require_object(w, "workload")
        _reject_unknown(w, "workload", ("mode", "n_items", "batch_size", "lr", "checkpointing"))
        cfg.workload.mode = _get(w, "workload", "mode", str, cfg.workload.mode)
        cfg.workload.n_items = _get(w, "workload", "n_items", int, cfg.workload.n_items)
        cfg.workload.batch_size = _get(w, "workload", "batch_size", int, cfg.workload.batch_size)
        cfg.workload.lr = float(np.float32(_get(w, "workload", "lr", float, cfg.workload.lr)))
        cfg.workload.checkpointing = _get(w, "workload", "checkpointing", bool, False)
    if "strategy" in j:
        s = j["strategy"]
        _require_object(s, "strategy")
        _reject_unknown(s, "strategy", ("kind", "k", "k_prime", "transfer_mode"))
        kind = _get(s, "strategy", "kind", str, "standard")
        if kind not in KIND_NAMES:
            raise ConfigError(f"config: unknown strategy kind '{kind}'")
        mode = _get(s, "strategy", "transfer_mode", str, "batch")
        if mode not in MODE_NAMES:
            raise ConfigError(f"config: unknown transfer_mode '{mode}'")
        cfg.strategy = E.StrategyConfig(KIND_NAMES[kind], _get(s, "strategy", "k", int, 0),
                                        _get(s, "strategy", "k_prime", int, 0), MODE_NAMES[mode])
    if "output" in j:
        o = j["output"]
        _require_object(o, "output")
        _reject_unknown(o, "output", ("dir", "formats"))
        if "dir" in o:
            cfg.output.dir = _get(o, "output", "dir", str, "out")
        cfg.output.formats = _get(o, "output", "formats", "strlist", cfg.output.formats)
    if "sweep" in j:
        s = j["sweep"]
        _require_object(s, "sweep")
        _reject_unknown(s, "sweep", ("k_min", "k_max", "k_prime_min", "k_prime_max",
                                     "budget_bytes", "objective"))
        spec = tuner.SweepSpec()
        spec.k_min = _get(s, "sweep", "k_min", int, spec.k_min)
        spec.k_max = _get(s, "sweep", "k_max", int, spec.k_max)
        spec.k_prime_min = _get(s, "sweep", "k_prime_min", int, spec.k_prime_min)
        spec.k_prime_max = _get(s, "sweep", "k_prime_max", int, spec.k_prime_max)
        spec.budget_bytes = _get(s, "sweep", "budget_bytes", "u64", 0)
        obj = _get(s, "sweep", "objective", str, "min_time_under_budget")
        if obj not in OBJECTIVES:
            raise ConfigError(f"config: unknown objective '{obj}'")
        spec.objective = OBJECTIVES[obj]
        cfg.sweep = spec
    return cfg


def load_config(path: str) -> ExperimentConfig:
    """experiment.cpp:140-216."""
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError as e:
        raise ConfigError(f"config: cannot open '{path}'") from e
    try:
        j = json.loads(raw)
    except ValueError as e:
        raise ConfigError(f"config: parse error in '{path}': {e}") from e
    return parse_config(j)


def output_dir(cfg: ExperimentConfig) -> str:
    """experiment.cpp:218-222."""
    if cfg.output.dir is not None:
        return cfg.output.dir
    env = os.environ.get("PIPESIM_OUTPUT_DIR")
    return env if env else "out"


# ---- execution ----------------------------------------------------------------------------

@dataclass
class ExperimentRun:
    summary: dict
    rows: list          # reference TraceEvent rows (trace_io.trace_rows)
    outputs: list = field(default_factory=list)
    loss: float | None = None


def execute(cfg: ExperimentConfig, strategy: E.StrategyConfig, numerics=E.EXACT) -> ExperimentRun:
    """experiment.cpp:84-101 on the GPU executor (inputs: make_input tags as the reference)."""
    m, w = cfg.model, cfg.workload
    model = E.build_model(m.seed, m.n_layers, m.d, m.frozen_prefix)
    strategy.validate(m.n_layers)
    train = w.mode == "train"
    with E.Executor(m.n_layers, m.d, strategy, numerics=numerics,
                    checkpointing=train and w.checkpointing,
                    capacity_bytes=cfg.arena.capacity_bytes, trace=True) as ex:
        ex.register_model(model)
        if train:
            x = E.make_input(m.seed, 0, w.batch_size, m.d)
            t = E.make_input(m.seed, 1, w.batch_size, m.d)
            loss = ex.train_step(x, t, w.lr)
            outputs = []
        else:
            xs = np.stack([E.make_input(m.seed, i, w.batch_size, m.d) for i in range(w.n_items)])
            outputs = list(ex.forward(xs))
            loss = None
        s = ex.stats()
        s["output_digest"] = ex.digest_train(loss) if train else E.digest_tensors(outputs)
        s.update(strategy=KIND_OF[strategy.kind], k=strategy.k, k_prime=strategy.k_prime)
        if train:
            s["has_loss"], s["loss"] = True, loss
        act_bytes = w.batch_size * m.d * 4
        rows = trace_io.trace_rows(ex, model.layer_bytes(), act_bytes)
    return ExperimentRun(summary=s, rows=rows, outputs=outputs, loss=loss)


def summary_line(s: dict) -> str:
    """print_summary_line (experiment.cpp:103-110); times are measured seconds."""
    line = (f"strategy={s['strategy']} k={s['k']} k_prime={s['k_prime']} peak_bytes={s['peak_bytes']} "
            f"per_item_time={trace_io.format_double(s['per_item_ms'] * 1e-3)} "
            f"stall={trace_io.format_double(s['stall_ms'] * 1e-3)} digest={s['output_digest']}")
    if s.get("has_loss"):
        line += f" loss={trace_io.format_double(float(np.float32(s['loss'])))}"
    return line


def _prepare(cfg):
    d = output_dir(cfg)
    os.makedirs(d, exist_ok=True)
    return d


def _write(path, body):
    with open(path, "w", newline="\n") as f:
        f.write(body)


def cmd_run(cfg: ExperimentConfig, numerics=E.EXACT, out=sys.stdout, err=sys.stderr) -> int:
    """experiment.cpp:224-243: 0, or 3 on OomDeadlockError (no artifacts written)."""
    cfg.validate()
    try:
        r = execute(cfg, cfg.strategy, numerics)
    except E.OomDeadlockError as e:
        print(f"error: {_message(e)}", file=err)
        return 3
    d = _prepare(cfg)
    if "csv" in cfg.output.formats:
        trace_io.export_trace_csv(r.rows, os.path.join(d, "trace.csv"))
    if "json" in cfg.output.formats:
        _write(os.path.join(d, "summary.json"), trace_io.summary_to_json(r.summary) + "\n")
    print(summary_line(r.summary), file=out)
    return 0


def cmd_compare(cfg: ExperimentConfig, numerics=E.EXACT, out=sys.stdout, err=sys.stderr) -> int:
    """experiment.cpp:245-291: the four strategies in fixed order on the configured window."""
    cfg.validate()
    sp_cfg = E.StrategyConfig(E.SUPERPIPELINE, cfg.strategy.k, cfg.strategy.k_prime,
                              cfg.strategy.transfer_mode)
    try:
        sp_cfg.validate(cfg.model.n_layers)
    except E.InvalidArgument as e:
        raise ConfigError(f"config: {_message(e)}") from e
    rows = []
    for kind in (E.STANDARD, E.CPU_ONLY, E.NAIVE, E.SUPERPIPELINE):
        s = E.StrategyConfig(kind, sp_cfg.k, sp_cfg.k_prime, sp_cfg.transfer_mode)
        if kind == E.CPU_ONLY:  # no GPU path: the ledger admits no weight, nothing is timed
            rows.append(dict(strategy="cpu_only", k=s.k, k_prime=s.k_prime, peak_bytes=0,
                             per_item_ms=math.nan, stall_ms=math.nan, output_digest=""))
            continue
        try:
            rows.append(execute(cfg, s, numerics).summary)
        except E.OomDeadlockError as e:
            print(f"error: {KIND_OF[kind]}: {_message(e)}", file=err)
            return 3
    timed = [r for r in rows if r["strategy"] != "cpu_only"]
    for r in timed:
        if r["output_digest"] != timed[0]["output_digest"]:
            print(f"error: digest mismatch between {timed[0]['strategy']} and {r['strategy']}", file=err)
            return 4
    csv = "Method,PeakBytes,PerItemTime,K,K'\n"
    for r in rows:
        csv += (f"{r['strategy']},{r['peak_bytes']},{trace_io.format_double(r['per_item_ms'] * 1e-3)},"
                f"{r['k']},{r['k_prime']}\n")
        if r["strategy"] != "cpu_only":
            print(summary_line(r), file=out)
    d = _prepare(cfg)
    if "csv" in cfg.output.formats:
        _write(os.path.join(d, "compare.csv"), csv)
    return 0


def cmd_sweep(cfg: ExperimentConfig, numerics=E.EXACT, repeats=3, out=sys.stdout,
              err=sys.stderr) -> int:
    """experiment.cpp:293-325: the (k, k') grid, each point measured on the GPU."""
    cfg.validate()
    if cfg.sweep is None:
        raise ConfigError("config: sweep section required for the sweep command")
    m, w = cfg.model, cfg.workload
    model = E.build_model(m.seed, m.n_layers, m.d, m.frozen_prefix)
    workload = tuner.SweepWorkload(n_items=w.n_items, batch_size=w.batch_size,
                                   transfer_mode=cfg.strategy.transfer_mode,
                                   train=w.mode == "train", lr=w.lr)
    try:
        evaluate = tuner.gpu_evaluator(model, workload, numerics=numerics, repeats=repeats,
                                       capacity_bytes=cfg.arena.capacity_bytes)
        result = tuner.grid_search(model, cfg.arena, workload, cfg.sweep, evaluate)
    except E.InvalidArgument as e:
        raise ConfigError(f"config: {_message(e)}") from e
    csv = "k,k_prime,feasible,peak_bytes,per_item_time\n"
    for e in result.table:
        csv += (f"{e.k},{e.k_prime},{1 if e.feasible else 0},{e.peak_bytes},"
                f"{trace_io.format_double(e.per_item_time)}\n")
    d = _prepare(cfg)
    if "csv" in cfg.output.formats:
        _write(os.path.join(d, "sweep.csv"), csv)
    if result.best:
        print(f"best k={result.best[0]} k_prime={result.best[1]}", file=out)
    else:
        print("none feasible", file=out)
    return 0


COMMANDS = {"run": cmd_run, "train": cmd_run, "compare": cmd_compare, "sweep": cmd_sweep}


def run_command(name: str, config, err=sys.stderr, **kwargs) -> int:
    """main.cpp:160-178 exit-code mapping around a command: ConfigError (and unknown commands)
    -> 2, OomDeadlockError -> 3, any other failure -> 1."""
    try:
        if name not in COMMANDS:
            raise ConfigError(f"unknown command '{name}'")
        cfg = config if isinstance(config, ExperimentConfig) else load_config(config)
        return COMMANDS[name](cfg, err=err, **kwargs)
    except ConfigError as e:
        print(f"error: {e}", file=err)
        return 2
    except E.OomDeadlockError as e:
        print(f"error: {_message(e)}", file=err)
        return 3
    except Exception as e:  # noqa: BLE001 - the reference maps std::exception to 1
        print(f"error: {e}", file=err)
        return 1
