"""bench.py's JSON line keeps the driver's contract (a small config, one GPU):
the base keys, `e2e` with its copied bytes, `roofline` with the dominant
kernel's achieved / peak / frac, `clocks`, `gpu_launches` and the accuracy
check of the emulated-FP64 factorization."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_bench_line_contract():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", "cfg1", "--steps", "5", "--warmup", "3",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "clocks", "gpu_launches"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 5 and line["warmup"] >= 3
    assert line["value"] > 0 and line["higher_is_better"] is True and line["dtype"] == "f64"
    assert "workload" in line["config"]
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["unit"] == line["unit"]
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    rf = line["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf, k
    assert rf["achieved"] > 0 and rf["peak"] > 0 and abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert line["gpu_launches"] > 0
    assert line["clocks"]["sm_mhz"] > 0
    acc = line["cholesky_accuracy"]
    assert acc["int8_emulated_vs_lapack_max_rel"] <= 1e-12 and acc["fp64_dmma_vs_lapack_max_rel"] <= 1e-12
