"""the Ada-Grouper decisions taken on the B200s are reproduced
bit-for-bit on the CPU — by the spec oracle and by the C++ decision function —
from the int64-ns compute/link samples the GPU run recorded.

Fixtures: tests/golden/gpu_tuner_log_*.json, written by bench.py --tuner-log on B200s:
  * n2_bursty (round 1): 2 stages, bursty ON/OFF trace, 5 rounds, no switch;
  * n4_square (round 2): 4 stages, square-wave trace (1.2 s preempted to 10 % of 400 Gb/s / 1.2 s
    free), re-tuned every 2 steps with passive link samples, 15 rounds; its first round switches
    from the warm-up incumbent k=1 to k=4 on the measured samples;
  * n4_square_cap16 (round 2): the same trace under a 16 GB cap ((k, b) frontier
    (1,4) (2,2) (3,1) (4,1)), 15 rounds;
  * n4_mixed (round 2): global batch 60 (M=30 at b=2) with the remainder-first mixed-k candidates;
    its first round switches to groups [2, 4×7] (chosen_groups), which the bench then ran.
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


def test_a_gpu_fixture_switches_to_a_mixed_plan():
    """A recorded GPU decision chose a mixed-k plan (group sizes) from group_candidates."""
    assert any(r["decision"].get("chosen_groups") and r["decision"]["switched"]
               for p in LOGS for r in json.loads(p.read_text())["rounds"])


def test_a_gpu_fixture_contains_a_switch():
    """At least one recorded GPU decision is a switch, so the replay covers switching, not only
    staying."""
    assert any(r["decision"]["switched"] for p in LOGS for r in json.loads(p.read_text())["rounds"])
