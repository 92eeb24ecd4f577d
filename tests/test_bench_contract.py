"""bench.py's JSON contract: both arms print ONE line with the same metric,
unit and config; ours carries value/e2e/roofline/clocks/gpu_launches (GPU
test), the reference arm its CPU baseline (CPU test, needs oracle/_ref)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling", "vs_baseline",
        "dtype", "data", "config", "e2e"}


def _run(*args, timeout=600):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line(refmod):
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "1", "--cpu-n", "8")
    assert BASE <= d.keys() and d["impl"] == "reference"
    baseline = json.loads((ROOT / "BASELINE.json").read_text())
    assert d["metric"] == baseline["metric"] and d["unit"] == "DOF-updates/s"
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["config"]["elements"] == 6 * 88 ** 3 and d["config"]["p"] == 4


@pytest.mark.gpu
def test_our_arm_line_matches_the_reference_arm(gpu_lib):
    d = _run("--cube-n", "16", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--curved-n", "8")
    assert BASE <= d.keys() and "impl" not in d
    assert d["metric"] == json.loads((ROOT / "BASELINE.json").read_text())["metric"]
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["warmup"] >= 3
    assert d["gpu_launches"] > 0 and d["dtype"] == "f64"
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and 0 < r["frac"] < 1
    assert abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
    c = d["curved"]  # the curved (isoparametric) path: its own value and roofline
    assert c["curved_elements"] == c["elements"] == 6 * 8 ** 3 and c["value"] == c["llf"]["value"] > 0
    for rm in ("llf", "hllc"):
        assert 0 < c[rm]["roofline"]["frac"] < 1 and c[rm]["rhs_kernel_ms"] > 0
    ref_cfg = _run("--impl", "reference", "--cube-n", "16", "--steps", "1", "--warmup", "1", "--cpu-n", "8")["config"]
    assert ref_cfg == d["config"]
