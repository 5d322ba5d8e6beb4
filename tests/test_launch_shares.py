"""scripts/launch_shares.py summarises the committed ncu launch list (profiles/) into a share table."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_launch_shares_on_committed_launch_list():
    out = subprocess.run([sys.executable, str(ROOT / "scripts/launch_shares.py"),
                          str(ROOT / "profiles/r1_launches_head.csv"), "--top", "3"],
                         capture_output=True, text=True, check=True).stdout
    assert out.startswith("4000 launches")
    rows = [ln for ln in out.splitlines() if ln.startswith("| gemm_bf16_2sm_kernel")]
    assert len(rows) == 3  # the three GEMM instantiations lead the step
    assert abs(sum(float(r.split("|")[4].strip().rstrip("%")) for r in rows) - 76.7) < 0.2
