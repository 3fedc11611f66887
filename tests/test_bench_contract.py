"""The driver's bench contract pieces that run without a GPU: the reference arm (the
reference's own CPU train step, oracle/_ref) prints one JSON line with the required keys, and
ranks other than 0 of a torchrun launch exit 0 without work."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra, *args):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                           "--model", "dense", "--layers", "2", "--d", "64", "--steps", "1", "--warmup", "0",
                           *args],
                          capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)


def test_reference_arm_prints_one_contract_line():
    r = _run({})
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "reference"


def test_reference_arm_other_ranks_exit_quietly():
    r = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, "--gpus", "2")
    assert r.returncode == 0, r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


def test_gpus_flag_without_torchrun_spawns_that_many_ranks():
    # `python bench.py --gpus 2` re-launches itself under torch.distributed.run with 2 ranks
    # (dry run: print the launch instead of running it)
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    env["SP_BENCH_DRY_SPAWN"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    cmd = json.loads(r.stdout.strip().splitlines()[-1])["spawn"]
    assert "torch.distributed.run" in cmd and "--nproc-per-node=2" in cmd
    assert "127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "2", "--steps", "1"]


def test_gpus_flag_must_match_the_torchrun_world():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env=dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0"))
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stdout


import pytest  # noqa: E402


@pytest.mark.gpu
def test_gpu_bench_line_has_every_contract_key():
    """bench.py on a small model (N = 1): one JSON line carrying the driver contract's keys,
    the roofline and e2e objects, our kernel launch count and the clock sample."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--model", "dense", "--layers", "6",
                        "--d", "256", "--rows", "1024", "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks", "north_star", "variants", "peak_hbm_gb"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["gpu_launches"] > 0
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * 1024 * 256 * 4
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] == 1
    assert set(d["variants"]) == {"adamw", "tf32"}
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
def test_gpu_bench_named_shape_line():
    """The default workload's code path (GPT-2 XL transformer layers) on a short stack: one
    contract line with the named-shape config, the in-step GEMM roofline, the HBM comparison
    against Standard and activation offload, and the FLOP-equivalent reference CPU baseline."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--layers", "4", "--seqs", "2",
                        "--k", "2", "--kp", "1", "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["config"]["model"] == "gpt2-xl" and d["config"]["params_per_layer"] > 30e6
    assert d["config"]["rows_per_gpu"] == 2048 and d["value"] > 0
    assert d["roofline"]["achieved"] > 0 and d["roofline"]["gemm_launches_per_step"] > 0
    assert set(d["variants"]) == {"adamw", "offload", "standard"}
    assert d["peak_hbm_gb"]["standard_measured_reserved"] > d["peak_hbm_gb"]["offload_measured_reserved"]
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * 2048 * 1600 * 4
    assert d["north_star"]["traced_step"]["attn_launches"] > 0
