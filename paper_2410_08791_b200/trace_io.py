"""Measured GPU timelines in the reference's trace formats.

The executor records one CUDA-event interval per op (sp_config.trace >= 1). Joined with the
op plan of the same call (Executor.last_plan(): layers moved, pass, ledger snapshot), each row
becomes a reference TraceEvent (trace.hpp:20-50), so the reference's tooling reads GPU runs:
  export_trace_csv   trace.cpp:144-155  header "t_start,t_end,kind,detail,resident_bytes,..."
  export_trace_json  trace.cpp:157-166  {"events": [...], "summary": {...}}
  import_trace_csv   trace.cpp:168-217  (strict header, detail key=value;... fields)
  summary_to_json    trace.cpp:219-237
Times are seconds of device time (the reference's are virtual seconds); numbers use the
shortest round-trip decimal form (format_double, trace.cpp:112-117 == Python repr).
"""
from __future__ import annotations

import json

HEADER = "t_start,t_end,kind,detail,resident_bytes,weight_bytes,activation_bytes,gradient_bytes"
_LIST_KEYS = ("layers", "slots", "w", "a", "o", "deps", "led")


def plan_ops(text: str):
    """Parses sp_describe_plan / sp_last_plan text into (header dict, list of op dicts)."""
    lines = text.strip().splitlines()
    head = dict(kv.split("=") for kv in lines[0].split() if "=" in kv)
    ops = []
    for ln in lines[1:]:
        parts = ln.split()
        op = {"index": int(parts[0]), "kind": parts[1]}
        for kv in parts[2:]:
            k, v = kv.split("=")
            if k == "md":  # per-move dependency lists: a.b|c|
                op[k] = [[int(t) for t in g.split(".") if t] for g in v.split("|")] if v else []
            elif k in _LIST_KEYS:
                op[k] = [int(t) for t in v.split(",")] if v else []
            else:
                op[k] = int(v) if v else None
        ops.append(op)
    return head, ops


def format_double(v: float) -> str:
    r = repr(float(v))
    return r[:-2] if r.endswith(".0") and "e" not in r else r


def _detail(row: dict) -> str:
    k = row["kind"]
    if k == "Compute":
        s = f"item={row['item']};layer={row['layer']};pass={'bwd' if row['backward'] else 'fwd'}"
        if row.get("compute_activation_bytes"):
            s += f";ab={row['compute_activation_bytes']}"
        if row.get("compute_gradient_bytes"):
            s += f";gb={row['compute_gradient_bytes']}"
        return s
    if k in ("H2D", "D2H"):
        s = "layers=" + "+".join(str(x) for x in row["layers"]) + f";wb={row['moved_weight_bytes']}"
        if row.get("moved_activation_bytes"):
            s += f";ab={row['moved_activation_bytes']}"
        return s
    return f"reason={row.get('reason', 'residency')}"


def trace_rows(executor, layer_bytes: int, act_bytes: int):
    """Reference TraceEvent rows (dicts) for the executor's last call."""
    head, ops = plan_ops(executor.last_plan())
    train = any(o["kind"] == "LOSS" for o in ops)
    ckpt = any(o["kind"] == "ACTSAVE" for o in ops)
    trainable = {o["layer"] for o in ops if o["kind"] == "UPDATE"}
    rows = []
    pending_stall = None
    for ev in executor.trace():
        if ev["kind"] == "Stall":
            pending_stall = ev
            continue
        op = ops[ev["op_index"]]
        if op.get("deferred"):
            continue  # this write-back runs at the start of the next call (its own row there)
        led = op.get("led", [0, 0, 0])
        row = {"t_start": ev["t_start"] * 1e-3, "t_end": ev["t_end"] * 1e-3,
               "weight_bytes": led[0], "activation_bytes": led[1], "gradient_bytes": led[2]}
        if op["kind"] == "COMPUTE":
            bwd = op.get("pass") == 1
            row.update(kind="Compute", item=op["item"], layer=op["layer"], backward=bwd,
                       compute_activation_bytes=(act_bytes if train and (not bwd or ckpt) else 0),
                       compute_gradient_bytes=(layer_bytes if bwd and op["layer"] in trainable else 0))
        elif op["kind"] in ("H2D", "D2H"):
            w = op.get("w", [])
            a = op.get("a", [])
            row.update(kind=op["kind"], layers=op.get("layers", []),
                       moved_weight_bytes=layer_bytes * sum(w),
                       moved_activation_bytes=act_bytes * sum(a))
        elif op["kind"] == "ACTSAVE":
            row.update(kind="D2H", layers=[op["layer"]], moved_weight_bytes=0,
                       moved_activation_bytes=act_bytes)
        else:
            continue
        if pending_stall is not None:
            rows.append({"t_start": pending_stall["t_start"] * 1e-3,
                         "t_end": pending_stall["t_end"] * 1e-3, "kind": "Stall",
                         "reason": "residency", "weight_bytes": led[0],
                         "activation_bytes": led[1], "gradient_bytes": led[2]})
            pending_stall = None
        rows.append(row)
    for r in rows:
        r["detail"] = _detail(r)
        r["resident_bytes"] = r["weight_bytes"] + r["activation_bytes"] + r["gradient_bytes"]
    return rows


def export_trace_csv(rows, path: str) -> None:
    with open(path, "w", newline="\n") as f:
        f.write(HEADER + "\n")
        for r in rows:
            f.write(",".join([format_double(r["t_start"]), format_double(r["t_end"]), r["kind"],
                              r["detail"], str(r["resident_bytes"]), str(r["weight_bytes"]),
                              str(r["activation_bytes"]), str(r["gradient_bytes"])]) + "\n")


def import_trace_csv(path: str):
    with open(path) as f:
        lines = f.read().splitlines()
    if not lines:
        raise RuntimeError(f"import_trace: '{path}' is empty")
    if lines[0] != HEADER:
        raise RuntimeError(f"import_trace: unexpected header in '{path}'")
    rows = []
    for line in lines[1:]:
        if not line:
            continue
        cols = line.split(",", 7)
        if len(cols) < 8:
            raise RuntimeError(f"import_trace: short row in '{path}'")
        r = {"t_start": float(cols[0]), "t_end": float(cols[1]), "kind": cols[2],
             "detail": cols[3], "resident_bytes": int(cols[4]), "weight_bytes": int(cols[5]),
             "activation_bytes": int(cols[6]), "gradient_bytes": int(cols[7])}
        if r["kind"] not in ("Compute", "H2D", "D2H", "Stall"):
            raise RuntimeError(f"trace: unknown event kind '{r['kind']}'")
        for field in cols[3].split(";"):
            key, _, value = field.partition("=")
            if key == "layers":
                r["layers"] = [int(v) for v in value.split("+")] if value else []
            elif key in ("item", "layer"):
                r[key] = int(value)
            elif key == "pass":
                r["backward"] = value == "bwd"
            elif key in ("wb", "ab", "gb"):
                r[key] = int(value)
            elif key == "reason":
                r["reason"] = value
            else:
                raise RuntimeError(f"import_trace: unknown detail key '{key}'")
        rows.append(r)
    return rows


def summary_to_json(s: dict) -> str:
    """trace.cpp:219-237 key order (times are measured seconds)."""
    out = {"strategy": s.get("strategy", ""), "k": s.get("k", 0), "k_prime": s.get("k_prime", 0),
           "peak_bytes": s["peak_bytes"], "per_item_time": s.get("per_item_ms", 0.0) * 1e-3,
           "makespan": s.get("makespan_ms", 0.0) * 1e-3,
           "total_stall_time": s.get("stall_ms", 0.0) * 1e-3,
           "n_transfers_h2d": s["n_transfers_h2d"], "n_transfers_d2h": s["n_transfers_d2h"],
           "output_digest": s.get("output_digest", ""),
           "peak_weight_bytes": s["peak_weight_bytes"],
           "peak_activation_bytes": s["peak_activation_bytes"],
           "peak_gradient_bytes": s["peak_gradient_bytes"],
           "total_gradient_bytes": s["total_gradient_bytes"]}
    if s.get("has_loss"):
        out["loss"] = s["loss"]
    return json.dumps(out, separators=(",", ":"))


def export_trace_json(rows, summary: dict, path: str) -> None:
    events = [{"t_start": r["t_start"], "t_end": r["t_end"], "kind": r["kind"],
               "detail": r["detail"], "resident_bytes": r["resident_bytes"],
               "weight_bytes": r["weight_bytes"], "activation_bytes": r["activation_bytes"],
               "gradient_bytes": r["gradient_bytes"]} for r in rows]
    with open(path, "w") as f:
        json.dump({"events": events, "summary": json.loads(summary_to_json(summary))}, f, indent=2)
        f.write("\n")
