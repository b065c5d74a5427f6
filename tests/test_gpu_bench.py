"""bench.py keeps the driver's JSON contract (both arms), on a real GPU.

Runs the script the way the driver does (a short --steps/--warmup run) and
checks every key the contract names, plus the invariants between them."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(*args, timeout=900):
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=str(ROOT), capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_line_contract():
    pytest.importorskip("torch").cuda.is_available() or pytest.skip("no GPU")
    d = _run("--steps", "5", "--warmup", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["dtype"] == "f64" and d["vs_baseline"] is None and "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert 0.5 < r["frac"] < 1.05  # the headline kernel streams A near the HBM roofline
    c = d["cpu_baseline"]
    assert c["kind"] in ("port", "reference") and c["cores"] >= 1 and c["value"] > 0
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 8 * 2**20 * 257 and e["d2h_bytes_per_step"] > 0
    assert 0 < e["value"] < d["value"]  # host buffers cross PCIe
    assert d["gpu_launches"] == 5
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    s = d["solve"]
    assert s["solves_per_sec"] > 0 and s["qr_solve_ms"] > 0 and s["sap_iterations"] > 0


def test_reference_arm_contract():
    d = _run("--impl", "reference", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["metric"].startswith("S·A sketch GB/s (config 2")
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["warmup"] == 3  # clamped to >= 3 like the GPU arm
