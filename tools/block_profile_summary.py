"""Writes the round's profiles/ summaries of a named-shape training step from ncu artifacts:

  python tools/block_profile_summary.py RAW.csv OUT.txt TRAFFIC.json "command line"

RAW.csv is `ncu -i REPORT --page raw --csv` of a `--set full` capture of one step of
tools/block_profile.py (every kernel of the step, in launch order). OUT.txt gets one block of key
metrics per launch (time, SM clock, tensor-pipe / MUFU / issue activity, DRAM bytes);
TRAFFIC.json the per-launch DRAM traffic of the step's tcgen05 GEMMs next to their algorithmic
bytes (operands read once + outputs written once), which bench.py reports as roofline.traffic."""
import csv
import json
import sys

METRICS = [
    ("time_us", "gpu__time_duration.sum", 1e-3),
    ("sm_ghz", "sm__cycles_elapsed.avg.per_second", 1.0),
    ("tensor_active_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("xu_inst_pct", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1.0),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    ("dram_read_mb", "dram__bytes_read.sum", 1.0),
    ("dram_write_mb", "dram__bytes_write.sum", 1.0),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct", 1.0),
    ("grid", "launch__grid_size", 1.0),
    ("regs", "launch__registers_per_thread", 1.0),
]


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def main(raw, out_txt, out_json, cmd):
    rows = list(csv.reader(open(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    lines = [f"ncu --set full --clock-control none --import-source on, one step of: {cmd}",
             "per launch, in launch order (serialised replay; clocks as the board ran them)", ""]
    gemm_bytes, gemm_names = [], []
    for r in data:
        name = r[col["Kernel Name"]]
        vals = {}
        for key, m, scale in METRICS:
            if m not in col:
                continue
            v = num(r[col[m]])
            if v is None:
                continue
            unit = units[col[m]]
            if m.startswith("dram__bytes"):
                v = v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1e-6)
            elif m == "gpu__time_duration.sum":
                v = v * {"nsecond": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
            elif m == "sm__cycles_elapsed.avg.per_second":
                v = v * {"Ghz": 1.0, "Mhz": 1e-3, "hz": 1e-9}.get(unit, 1.0)
            vals[key] = v
        short = name.split("(")[0]
        lines.append(short)
        lines.append("    " + "  ".join(f"{k}={v:.4g}" for k, v in vals.items()))
        if "gemm" in short and "dram_read_mb" in vals:
            gemm_bytes.append((vals["dram_read_mb"] + vals.get("dram_write_mb", 0.0)) * 1e6)
            gemm_names.append(short)
    open(out_txt, "w").write("\n".join(lines) + "\n")
    if gemm_bytes:
        # algorithmic bytes of the GPT-2 XL layer's 12 GEMMs at 16 x 1024 tokens (bf16 operands,
        # fp32 residual / gate / dX outputs, fp32 dW split partials as choose_dw writes them)
        T, d, ff, q = 16384, 1600, 6400, 4800
        b2, b4 = 2, 4
        algo = [
            T * d * b2 + d * q * b2 + T * q * b2,                          # QKV (+bias)
            T * d * b2 + d * d * b2 + 2 * T * d * b4,                      # Wo + residual (fp32 in / out)
            T * d * b2 + d * ff * b2 + 2 * T * ff * b2,                    # FC1 -> GELU out + pre-activation
            T * ff * b2 + ff * d * b2 + 2 * T * d * b4,                    # FC2 + residual
            T * ff * b2 + T * d * b2 + ff * d * b4,                        # dW2 (one fp32 image)
            T * d * b2 + ff * d * b2 + 2 * T * ff * b2,                    # dg = dy W2^T * gelu'(h)
            T * d * b2 + T * ff * b2 + d * ff * b4,                        # dW1
            T * ff * b2 + d * ff * b2 + T * d * b4,                        # dxn2 (fp32 out)
            T * d * b2 + T * d * b2 + d * d * b4,                          # dWo
            T * d * b2 + d * d * b2 + T * d * b2,                          # do
            T * d * b2 + T * q * b2 + d * q * b4,                          # dWqkv
            T * q * b2 + d * q * b2 + T * d * b4,                          # dxn1 (fp32 out)
        ]
        rec = {"kernel": "tcgen05 bf16 GEMMs of the GPT-2 XL block step (gemm2_kernel, all variants)",
               "bytes_per_launch": sum(gemm_bytes) / len(gemm_bytes),
               "algorithmic_bytes_per_launch": sum(algo) / len(algo),
               "launches_captured": len(gemm_bytes),
               "source": out_txt + " (dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged)"}
        json.dump(rec, open(out_json, "w"), indent=1)
        print(json.dumps(rec))


if __name__ == "__main__":
    main(*sys.argv[1:5])
