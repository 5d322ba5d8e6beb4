"""The C-ABI library loads on a CPU-only host and exports every symbol include/ptk.h declares."""
import ctypes
import re
from pathlib import Path

from paper_2303_01675_b200 import _lib as L

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "ptk.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ptk_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    lib = L.lib()
    names = declared_symbols()
    assert len(names) >= 10
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_version_and_error_channel():
    lib = L.lib()
    assert lib.ptk_version().startswith(b"ptk")
    # a planner call with a bad k fails with a typed status and a message
    from paper_2303_01675_b200 import pipetune as pt
    try:
        pt.plan_kfkb(pt.uniform_model(2, 4), 1, 9)
    except pt.PipetuneError as e:
        assert e.kind == "PlanError"
    assert b"k=9" in lib.ptk_last_error()


def test_no_cpu_fallback_symbols():
    """The product library has no host implementation of the stage math to fall back on."""
    out = ctypes.CDLL(str(L.LIB_PATH))
    for sym in ("ptk_stage_forward_cpu", "ptk_gemm_cpu"):
        assert not hasattr(out, sym)
