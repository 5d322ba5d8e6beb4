"""C++ callers of the drop-in API: examples/cpp_api_demo.cpp (reference planner calls + the spec-module
extensions: simulate over a preempted link, mixed-k tuning_round_plans, result_from_records) compiles
against include/pipetune and libptk.so and prints the expected decisions."""
import shutil
import subprocess
from pathlib import Path

import pytest

from paper_2303_01675_b200 import _lib as L

ROOT = Path(__file__).resolve().parents[1]


def test_cpp_api_demo(tmp_path):
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    exe = tmp_path / "demo"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(ROOT / "examples" / "cpp_api_demo.cpp"),
                    f"-L{L.LIB_PATH.parent}", "-lptk", f"-Wl,-rpath,{L.LIB_PATH.parent}", "-o", str(exe)],
                   check=True, capture_output=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines()
    assert out[0].startswith("stage 0: F0 F1 F2 F3")           # kFkB k=4 warm-up on stage 0 (S=4, M=10)
    assert "chosen k=4 groups=3 switched=1" in out[2]           # remainder-first [2, 4, 4] wins over uniform k=4
    assert out[3] == "records reproduce: 1"
