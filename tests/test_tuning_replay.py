"""the Ada-Grouper decisions taken on the B200s are reproduced
bit-for-bit on the CPU — by the spec oracle and by the C++ decision function —
from the int64-ns compute/link samples the GPU run recorded.

Fixture: tests/golden/gpu_tuner_log_*.json, written by
  torchrun --nproc-per-node 2 bench.py --gpus 2 --trace two-regime --retune 2 --tuner-log ...
on 2x B200 (round 1).
"""
import copy
import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import spec_oracle as O  # noqa: E402
from paper_2303_01675_b200 import pipetune as pt  # noqa: E402

LOGS = sorted((ROOT / "tests" / "golden").glob("gpu_tuner_log_*.json"))


@pytest.mark.parametrize("path", LOGS, ids=[p.stem for p in LOGS])
def test_gpu_decisions_replay_bit_exact(path):
    log = json.loads(path.read_text())
    assert log["rounds"], "empty tuner log"
    ks = []
    for rnd in log["rounds"]:
        req, got = rnd["request"], rnd["decision"]
        assert O.run(copy.deepcopy(req))["decision"] == got
        assert pt.scenario(req)["decision"] == got
        ks.append(got["chosen"][0])
    assert all(k >= 1 for k in ks)
