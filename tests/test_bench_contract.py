"""bench.py's JSON contract (the driver parses it): one JSON line on stdout with every key, at N=1,
for our arm and for the reference arm.  BERT-large with a small global batch keeps it short."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline"}


def _run(args):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout  # exactly one line on stdout
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_line_has_every_key():
    d = _run(["--model", "bert-large", "--global-batch", "16", "--micro-batch", "4", "--steps", "3", "--warmup", "3"])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert set(d["roofline"]) >= {"bound", "achieved", "peak", "unit", "frac", "traffic"}
    assert 0 < d["roofline"]["frac"] < 1.2
    assert set(d["e2e"]) == {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"}
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["gpu_launches"] > 0
    assert set(d["cpu_baseline"]) >= {"value", "unit", "cores", "kind", "sample"}
    assert "workload" in d["config"] and "sm_mhz" in d["clocks"]


@pytest.mark.gpu
def test_reference_arm_line():
    d = _run(["--impl", "reference", "--model", "bert-large", "--steps", "1", "--warmup", "0"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
