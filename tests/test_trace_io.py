"""Reference trace formats for measured GPU timelines (trace.cpp:112-237): header, detail
strings, CSV round trip, summary JSON key order. CPU cases use synthetic rows; the GPU case
exports a real run and re-imports it."""
import json
import os

import numpy as np
import pytest

from paper_2410_08791_b200 import trace_io


def synthetic_rows():
    rows = [
        {"t_start": 0.0, "t_end": 1e-4, "kind": "H2D", "layers": [0, 1], "moved_weight_bytes": 2176,
         "moved_activation_bytes": 0, "weight_bytes": 2176, "activation_bytes": 64, "gradient_bytes": 0},
        {"t_start": 1e-4, "t_end": 1.5e-4, "kind": "Stall", "reason": "residency",
         "weight_bytes": 2176, "activation_bytes": 64, "gradient_bytes": 0},
        {"t_start": 1.5e-4, "t_end": 2e-4, "kind": "Compute", "item": 0, "layer": 0, "backward": False,
         "compute_activation_bytes": 64, "compute_gradient_bytes": 0,
         "weight_bytes": 2176, "activation_bytes": 128, "gradient_bytes": 0},
        {"t_start": 3e-4, "t_end": 4e-4, "kind": "Compute", "item": 0, "layer": 1, "backward": True,
         "compute_activation_bytes": 0, "compute_gradient_bytes": 1088,
         "weight_bytes": 2176, "activation_bytes": 128, "gradient_bytes": 1088},
        {"t_start": 4e-4, "t_end": 5e-4, "kind": "D2H", "layers": [1], "moved_weight_bytes": 1088,
         "moved_activation_bytes": 64, "weight_bytes": 1088, "activation_bytes": 64, "gradient_bytes": 0},
    ]
    for r in rows:
        r["detail"] = trace_io._detail(r)
        r["resident_bytes"] = r["weight_bytes"] + r["activation_bytes"] + r["gradient_bytes"]
    return rows


def test_detail_strings_match_reference_format():
    rows = synthetic_rows()
    assert rows[0]["detail"] == "layers=0+1;wb=2176"
    assert rows[1]["detail"] == "reason=residency"
    assert rows[2]["detail"] == "item=0;layer=0;pass=fwd;ab=64"
    assert rows[3]["detail"] == "item=0;layer=1;pass=bwd;gb=1088"
    assert rows[4]["detail"] == "layers=1;wb=1088;ab=64"


def test_csv_round_trip(tmp_path):
    rows = synthetic_rows()
    p = tmp_path / "trace.csv"
    trace_io.export_trace_csv(rows, str(p))
    text = p.read_text()
    assert text.splitlines()[0] == trace_io.HEADER
    back = trace_io.import_trace_csv(str(p))
    assert len(back) == len(rows)
    for a, b in zip(rows, back):
        assert a["t_start"] == b["t_start"] and a["t_end"] == b["t_end"] and a["kind"] == b["kind"]
        assert a["resident_bytes"] == b["resident_bytes"] and a["detail"] == b["detail"]
    assert back[0]["layers"] == [0, 1] and back[2]["backward"] is False


def test_import_rejects_bad_header(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("t_start,t_end,kind\n0,1,Compute\n")
    with pytest.raises(RuntimeError):
        trace_io.import_trace_csv(str(p))


def test_format_double_is_shortest_round_trip():
    for v in (0.0, 1e-4, 74.44, 1.0 / 3.0, 5.0):
        s = trace_io.format_double(v)
        assert float(s) == v
    assert trace_io.format_double(5.0) == "5"


def test_summary_json_key_order():
    s = {"strategy": "superpipeline", "k": 4, "k_prime": 2, "peak_bytes": 6592, "per_item_ms": 1.0,
         "makespan_ms": 2.0, "stall_ms": 0.5, "n_transfers_h2d": 15, "n_transfers_d2h": 0,
         "output_digest": "046c06b54d8304c5", "peak_weight_bytes": 6528, "peak_activation_bytes": 64,
         "peak_gradient_bytes": 0, "total_gradient_bytes": 0}
    keys = list(json.loads(trace_io.summary_to_json(s)).keys())
    assert keys == ["strategy", "k", "k_prime", "peak_bytes", "per_item_time", "makespan",
                    "total_stall_time", "n_transfers_h2d", "n_transfers_d2h", "output_digest",
                    "peak_weight_bytes", "peak_activation_bytes", "peak_gradient_bytes",
                    "total_gradient_bytes"]


@pytest.mark.gpu
def test_gpu_run_exports_reference_trace(tmp_path):
    import paper_2410_08791_b200 as sp
    model = sp.build_model(6, 8, 4)
    x, t = sp.make_input(6, 0, 4, 4), sp.make_input(6, 1, 4, 4)
    with sp.Executor(8, 4, sp.StrategyConfig(sp.SUPERPIPELINE, 3, 1), checkpointing=True, trace=1) as ex:
        ex.register_model(model)
        loss = ex.train_step(x, t, 0.01)
        st = ex.stats()
        rows = trace_io.trace_rows(ex, model.layer_bytes(), 4 * 4 * 4)
    p = tmp_path / "trace.csv"
    trace_io.export_trace_csv(rows, str(p))
    back = trace_io.import_trace_csv(str(p))
    kinds = [r["kind"] for r in back]
    assert kinds.count("Compute") == 16  # 8 forward + 8 backward
    assert kinds.count("H2D") == st["n_transfers_h2d"]
    assert max(r["resident_bytes"] for r in back) <= st["peak_bytes"]
    assert all(r["t_end"] >= r["t_start"] for r in back)
    trace_io.export_trace_json(rows, dict(st, has_loss=True, loss=loss, strategy="superpipeline",
                                          k=3, k_prime=1), str(tmp_path / "trace.json"))
    j = json.loads((tmp_path / "trace.json").read_text())
    assert len(j["events"]) == len(rows) and j["summary"]["loss"] == pytest.approx(loss)
