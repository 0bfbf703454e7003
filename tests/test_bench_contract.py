"""bench.py's one-line JSON contract: the reference arm (CPU, the reference
built from its sources in oracle/_ref) here, and our arm on the GPU.  Small
workloads: these check the keys and their meaning, not performance."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

import oracle

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout,
                         env={**os.environ, "PYTHONPATH": str(ROOT)})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


@pytest.mark.skipif(not oracle.available("reference"), reason="oracle/_ref not built")
def test_reference_arm_line():
    r = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0", "--elems", "3",
                  "--cpu-iters", "2")
    assert r["impl"] == "reference"
    assert BASE_KEYS <= set(r)
    assert r["unit"] == "GDOF/s" and r["higher_is_better"] is True and r["value"] > 0
    assert r["cpu_baseline"]["kind"] == "reference" and r["cpu_baseline"]["value"] == r["value"]
    assert r["e2e"] == {"value": r["value"], "unit": r["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_line():
    r = run_bench("--steps", "3", "--warmup", "3", "--elems", "6", "--no-cpu")
    assert BASE_KEYS | {"roofline", "gpu_launches", "clocks"} <= set(r)
    assert r["n_gpus"] == 1 and r["steps"] == 3 and r["warmup"] == 3 and r["value"] > 0
    assert r["dtype"] == "f64" and r["config"]["workload"].startswith("bp5 p=7")
    rf = r["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] <= 1.5
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    e = r["e2e"]
    n_vec = (6 * 7 + 1) ** 3
    assert e["h2d_bytes_per_step"] == 8 * n_vec and e["d2h_bytes_per_step"] == 8 * n_vec
    assert r["gpu_launches"] > 0


@pytest.mark.skipif(not oracle.available("reference"), reason="oracle/_ref not built")
def test_reference_arm_defaults_to_the_same_workload():
    r = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0", "--elems", "3")
    assert r["config"]["same_config"] is True
    assert "20 fixed iterations" in r["config"]["workload"]


@pytest.mark.gpu
def test_our_arm_verifies_its_timed_result():
    """With the CPU legs on, the line carries the cpu_baseline and the check of
    the timed step's residual history and iterate against the reference."""
    r = run_bench("--steps", "3", "--warmup", "3", "--elems", "5")
    v = r["verification"]
    assert v["ok"], v
    assert v["iterations"] == [20, 20]
    assert r["cpu_baseline"]["value"] > 0 and r["cpu_baseline"]["cores"] >= 1
    assert r["e2e"]["serial"]["value"] > 0


@pytest.mark.gpu
def test_group_emulation_runs_the_partitioned_path():
    """bench.py --group 2: the --gpus N code path (partition, exchange,
    all-reduce) on one GPU, checked against the single-domain solve."""
    r = run_bench("--group", "2", "--steps", "2", "--warmup", "1", "--elems", "4")
    assert r["emulated_ranks"] == 2 and r["value"] > 0
    assert r["verification"]["ok"], r["verification"]
