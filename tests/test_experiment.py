"""Experiment harness (paper_2410_08791_b200/experiment.py) against the reference's own
config tests (test_config.cpp) and shipped configs (tests/golden/configs, written by
tests/golden/make_golden.py from the reference's configs/)."""
import io
import json
import os

import numpy as np
import pytest

import paper_2410_08791_b200 as sp
from paper_2410_08791_b200 import experiment as X
from paper_2410_08791_b200 import trace_io

HERE = os.path.dirname(os.path.abspath(__file__))
CFG = os.path.join(HERE, "golden", "configs")
GOLD = {c["name"]: c for c in json.load(open(os.path.join(HERE, "golden", "golden.json")))["cases"]}


def write(tmp_path, name, body):
    p = tmp_path / name
    p.write_text(body)
    return str(p)


def test_default_config_loads_with_expected_values():  # test_config.cpp:43-58
    cfg = X.load_config(os.path.join(CFG, "default.json"))
    assert (cfg.model.seed, cfg.model.n_layers, cfg.model.d) == (7, 8, 16)
    assert cfg.arena.d2h_bandwidth == 100.0 and cfg.arena.h2d_bandwidth == 200.0
    assert cfg.workload.mode == "infer" and cfg.workload.n_items == 4
    assert cfg.strategy.kind == sp.SUPERPIPELINE and (cfg.strategy.k, cfg.strategy.k_prime) == (4, 2)
    assert cfg.sweep is not None and cfg.sweep.k_max == 8
    cfg.validate()
    train = X.load_config(os.path.join(CFG, "oom_train.json"))
    assert train.workload.mode == "train" and train.arena.capacity_bytes == 15000
    train.validate()


@pytest.mark.parametrize("body", ['{"modell": {}}', '{"model": {"layers": 4}}',
                                  '{"strategy": {"kind": "naive", "K": 2}}',
                                  '{"sweep": {"k_min": 2, "budget": 5}}'])
def test_unknown_keys_are_rejected_at_every_level(tmp_path, body):  # test_config.cpp:60-67
    with pytest.raises(X.ConfigError, match="unknown key"):
        X.load_config(write(tmp_path, "c.json", body))


@pytest.mark.parametrize("body", ['{"model": {"n_layers": "eight"}}', '{"strategy": {"kind": "turbo"}}',
                                  '{not json', '[1, 2]', '{"model": 3}',
                                  '{"workload": {"checkpointing": 1}}', '{"model": {"d": true}}',
                                  '{"output": {"formats": "csv"}}',
                                  '{"strategy": {"kind": "naive", "transfer_mode": "burst"}}',
                                  '{"sweep": {"objective": "fastest"}}'])
def test_malformed_values_are_config_errors(tmp_path, body):  # test_config.cpp:69-77
    with pytest.raises(X.ConfigError):
        X.load_config(write(tmp_path, "c.json", body))


def test_missing_file_is_config_error():
    with pytest.raises(X.ConfigError, match="cannot open"):
        X.load_config("missing_file.json")


def test_numbers_convert_like_the_reference(tmp_path):
    cfg = X.load_config(write(tmp_path, "c.json", '{"model": {"n_layers": 4.9, "seed": -1}}'))
    assert cfg.model.n_layers == 4 and cfg.model.seed == (1 << 64) - 1


def test_validation_enforces_cross_field_invariants():  # test_config.cpp:79-93
    def fresh():
        return X.load_config(os.path.join(CFG, "default.json"))
    for mutate in (lambda c: setattr(c.strategy, "k_prime", 4),
                   lambda c: setattr(c.workload, "mode", "predict"),
                   lambda c: setattr(c.model, "frozen_prefix", 9),
                   lambda c: setattr(c.output, "formats", ["yaml"]),
                   lambda c: setattr(c.workload, "lr", 0.0),
                   lambda c: setattr(c.arena, "h2d_bandwidth", 0.0),
                   lambda c: setattr(c.sweep, "budget_bytes", 0)):
        c = fresh()
        mutate(c)
        with pytest.raises(X.ConfigError):
            c.validate()


def test_output_dir_resolution(monkeypatch):  # test_config.cpp:95-104
    cfg = X.ExperimentConfig()
    monkeypatch.delenv("PIPESIM_OUTPUT_DIR", raising=False)
    assert X.output_dir(cfg) == "out"
    monkeypatch.setenv("PIPESIM_OUTPUT_DIR", "env_dir")
    assert X.output_dir(cfg) == "env_dir"
    cfg.output.dir = "explicit_dir"
    assert X.output_dir(cfg) == "explicit_dir"


def test_exit_codes_without_gpu_work(tmp_path):  # main.cpp:160-178
    err = io.StringIO()
    assert X.run_command("run", "does_not_exist.json", err=err) == 2
    assert X.run_command("frobnicate", os.path.join(CFG, "default.json"), err=err) == 2
    cfg = X.load_config(os.path.join(CFG, "default.json"))
    cfg.strategy.k_prime = 7  # invalid window: exit 2 and no artifacts
    cfg.output.dir = str(tmp_path / "bad")
    assert X.run_command("run", cfg, err=err) == 2
    assert not (tmp_path / "bad").exists()
    assert "error:" in err.getvalue()
    cfg = X.load_config(os.path.join(CFG, "default.json"))
    cfg.sweep = None
    assert X.run_command("sweep", cfg, err=err) == 2  # sweep needs its section


# ---- on the GPU: the commands themselves ----------------------------------------------------

@pytest.mark.gpu
def test_run_writes_reference_artifacts(tmp_path):  # test_config.cpp:106-114, 135-142
    out = io.StringIO()
    cfg = X.load_config(os.path.join(CFG, "default.json"))
    summaries = []
    for name in ("a", "b"):
        cfg.output.dir = str(tmp_path / name)
        assert X.cmd_run(cfg, out=out) == 0
        assert (tmp_path / name / "trace.csv").exists()
        summaries.append(json.loads((tmp_path / name / "summary.json").read_text()))
    line = out.getvalue().splitlines()[0]
    assert "strategy=superpipeline" in line and "digest=046c06b54d8304c5" in line
    g = GOLD["default.json/superpipeline"]
    for s in summaries:  # ledger and digest fields are deterministic (times are measured)
        assert s["output_digest"] == g["digest"] and s["peak_bytes"] == g["peak_bytes"]
        assert s["n_transfers_h2d"] == g["n_transfers_h2d"]
        assert list(s)[:3] == ["strategy", "k", "k_prime"]
    rows = trace_io.import_trace_csv(str(tmp_path / "a" / "trace.csv"))
    assert {r["kind"] for r in rows} >= {"Compute", "H2D"}


@pytest.mark.gpu
def test_train_config_completes_windowed_but_ooms_standard(tmp_path):  # test_config.cpp:166-175
    out, err = io.StringIO(), io.StringIO()
    cfg = X.load_config(os.path.join(CFG, "oom_train.json"))
    cfg.output.dir = str(tmp_path / "train")
    assert X.run_command("train", cfg, out=out, err=err) == 0
    assert "loss=" in out.getvalue() and "digest=44ab7f18e19ef8b8" in out.getvalue()
    s = json.loads((tmp_path / "train" / "summary.json").read_text())
    assert np.float32(s["loss"]).tobytes().hex() == GOLD["oom_train.json/superpipeline"]["loss_bits"]
    cfg.strategy = sp.StrategyConfig(sp.STANDARD)
    cfg.output.dir = str(tmp_path / "std")
    assert X.run_command("train", cfg, out=out, err=err) == 3
    assert not (tmp_path / "std" / "trace.csv").exists()


@pytest.mark.gpu
def test_compare_emits_four_strategy_table_in_fixed_order(tmp_path):  # test_config.cpp:144-160
    out = io.StringIO()
    cfg = X.load_config(os.path.join(CFG, "default.json"))
    cfg.output.dir = str(tmp_path)
    assert X.cmd_compare(cfg, out=out) == 0
    lines = (tmp_path / "compare.csv").read_text().splitlines()
    assert lines[0] == "Method,PeakBytes,PerItemTime,K,K'"
    assert [ln.split(",")[0] for ln in lines[1:]] == ["standard", "cpu_only", "naive", "superpipeline"]
    peaks = {ln.split(",")[0]: int(ln.split(",")[1]) for ln in lines[1:]}
    assert peaks["superpipeline"] == GOLD["default.json/superpipeline"]["peak_bytes"]
    assert peaks["standard"] == GOLD["default.json/standard"]["peak_bytes"]
    assert peaks["naive"] == GOLD["default.json/naive"]["peak_bytes"]
    assert peaks["cpu_only"] == 0
    assert out.getvalue().count("digest=046c06b54d8304c5") == 3


@pytest.mark.gpu
def test_sweep_writes_table_and_best_pair(tmp_path):  # test_config.cpp:162-164
    out = io.StringIO()
    cfg = X.load_config(os.path.join(CFG, "default.json"))
    cfg.sweep.k_max = 4
    cfg.output.dir = str(tmp_path)
    assert X.cmd_sweep(cfg, out=out, repeats=1) == 0
    assert (tmp_path / "sweep.csv").read_text().startswith("k,k_prime,feasible,peak_bytes,per_item_time\n")
    assert "best k=" in out.getvalue()
    cfg.sweep.budget_bytes = 10  # below one layer: exit 0, explicitly nothing feasible
    out = io.StringIO()
    assert X.cmd_sweep(cfg, out=out, repeats=1) == 0
    assert "none feasible" in out.getvalue()
