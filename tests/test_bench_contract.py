"""bench.py keeps the driver's JSON contract: our arm on the GPU, the
reference arm (the float64 oracle) on the host."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

BASE = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1", "--ref-step-seconds", "1"])
    assert BASE <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "elements/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--config", "c2", "--extra", "none"])
    assert BASE <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["dtype"] == "f64" and "workload" in d["config"] and "l2" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and r["peak"] > 0 and 0 < r["frac"] <= 1
    assert r["achieved"] > 0 and "traffic" in r
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["status_bits"] & 3 == 0
    # per-pass HBM evidence of the full-array kernels
    for k in ("pass_level_gram", "pass_project_x", "pass_project_w", "pass_expand"):
        assert d["hbm_passes"][k]["alg_GBps"] > 0
    assert d["t2"]["min_margin"] > 0
    # both arms describe the workload with the identical config dict
    ref = _run(["--impl", "reference", "--config", "c2", "--steps", "1", "--warmup", "1",
                "--ref-step-seconds", "1"])
    assert ref["config"] == d["config"]
    assert ref["metric"] == d["metric"] and ref["unit"] == d["unit"] and ref["scaling"] == d["scaling"]
