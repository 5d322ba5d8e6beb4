"""Pin the spec oracle (oracle/spec_oracle.py) to SPEC.md's examples and acceptance criteria.

The reference ships no code for these modules, so these
examples are the only pins; every value asserted here is quoted from SPEC.md.
"""
import sys
from pathlib import Path

import pytest

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import spec_oracle as O  # noqa: E402
from tests.spec_scenarios import const_traces, fig2, stage, zero_comm  # noqa: E402

U = O.TICKS


def test_compute_duration_examples():
    assert O.compute_ticks(stage(f=1.0, ff=0.0), 4, True) == 4 * U
    assert O.compute_ticks(stage(b=0.5, bf=1.0), 2, False) == 2 * U


def test_graph_counts():
    for S, M, want in ((1, 1, (1, 1, 0, 0, 1)), (2, 1, (2, 2, 2, 2, 2)), (4, 8, (32, 32, 48, 48, 4))):
        g = O.Graph([stage() for _ in range(S)], 1, M)
        kinds = [n[0] for n in g.nodes]
        assert tuple(kinds.count(k) for k in range(5)) == want


def test_peak_memory_examples():
    model = {"global_batch": 4, "stages": [stage(act=100), stage(act=100)]}
    st, g, orders, _ = O.make_plan(model, {"kind": "1f1b", "micro_batch_size": 1})
    assert O.peak_memory(st, g, orders)[0][0] == 200
    st, g, orders, _ = O.make_plan(model, {"kind": "gpipe", "micro_batch_size": 1})
    assert O.peak_memory(st, g, orders)[0][0] == 400
    m1 = {"global_batch": 1, "stages": [stage(act=100, w=7)]}
    st, g, orders, _ = O.make_plan(m1, {"kind": "1f1b", "micro_batch_size": 1})
    assert O.peak_memory(st, g, orders)[0] == [107]


def test_enumerate_synthetic_peak():
    out = O.enumerate_candidates({"global_batch": 40, "stages": [stage()]}, 1600, 3,
                                 feasible=lambda k, b: (k + 1) * b * 100 <= 1600)
    assert [(k, b) for k, b, _, _ in out] == [(1, 8), (2, 5), (3, 4)]


def test_enumerate_infinite_limit():  # only k=1 can take b=global_batch
    out = O.enumerate_candidates({"global_batch": 8, "stages": [stage(act=1)]}, 10**18, 3)
    assert out[0][:2] == (1, 8)
    assert all(b < 8 for k, b, _, _ in out[1:])


def test_transfer_duration_examples():
    tr = {"base_bandwidth": 10.0, "latency": 0.25, "segments": []}
    assert O.transfer_duration(tr, 0, 0) == U // 4
    assert O.transfer_duration({"base_bandwidth": 10.0, "latency": 0.0}, 100, 0) == 10 * U
    dip = {"base_bandwidth": 10.0, "latency": 0.0, "segments": [[0.0, 20.0, 0.5]]}
    assert O.transfer_duration(dip, 150, 0) == 25 * U


def test_estimate_examples():
    s = O.Store(2)
    s.record(0, 1, 2 * U)
    s.record(0, 1, 4 * U)
    assert s.estimate(0, 1) == 3 * U
    s = O.Store(2)
    for v in (1, 1, 1, 9):
        s.record(0, 1, v * U)
    assert s.estimate(0, 1) == 5 * U
    with pytest.raises(O.SpecError):
        O.Store(2).estimate(0, 1)


def test_simulate_examples():  # SPEC.md:348-349, 366 (acceptance 3)
    assert O.run(zero_comm(1, 4))["result"]["pipeline_length"] == 12 * U
    assert O.run(zero_comm(2, 2))["result"]["pipeline_length"] == 9 * U
    for S in range(1, 6):
        for M in range(S, 11):
            for kind in ("1f1b", "gpipe"):
                assert O.run(zero_comm(S, M, kind))["result"]["pipeline_length"] == (M + S - 1) * 3 * U


def test_fig2_acceptance_1():
    l1 = O.run(fig2(k=1))["result"]
    l2 = O.run(fig2(k=2))["result"]
    assert l2["pipeline_length"] <= 0.95 * l1["pipeline_length"]
    zero = O.run(fig2(k=1, xfer_bytes=0))["result"]
    assert max(l1["bubble_fraction"]) > max(zero["bubble_fraction"])
    assert all(a > b for a, b in zip(l1["bubble_fraction"], l2["bubble_fraction"]))


def test_queue_first_forward_not_prebuffered():
    r = O.run(zero_comm(2, 2))["result"]
    assert r["launches"][1][0][1] == 0


def test_rank_tie_break():
    assert O.decide([[2, 1, 4, 80], [1, 1, 4, 100]], None, 0.02)[0] == [2, 1, 4]
    ranked = sorted([[3, 1, 4, 50], [2, 1, 4, 50]], key=lambda e: (e[3], e[0], -e[1]))
    assert ranked[0][0] == 2


def test_tuner_zero_comm_never_switches():
    # "max-b" holds where the fixed per-launch cost is the only b-dependent term,
    # i.e. without a pipeline fill bubble (S=1); with S>1 smaller b shortens the fill.
    model = {"global_batch": 8, "stages": [stage(ff=0.5, bf=1.0, act=1)]}
    out = O.run({"op": "tune", "model": model, "cluster": {"device_memory_limit": 10**12, "devices": 1},
                 "traces": [], "policy": {"interval": 50.0, "k_max": 4}, "horizon": 400.0})
    assert not any(r["switched"] for r in out["rounds"])
    assert out["rounds"][0]["chosen"][1] == 8  # max-b candidate: best compute efficiency


def test_tuner_full_hysteresis_never_switches():
    model = {"global_batch": 8, "stages": [stage(out_f=5, out_b=5, act=1) for _ in range(3)]}
    tr = const_traces(3, base=10.0)
    for t in tr:
        t["segments"] = [[0.0, 200.0, 0.1]]
    out = O.run({"op": "tune", "model": model, "cluster": {"device_memory_limit": 10**12, "devices": 3},
                 "traces": tr, "policy": {"interval": 30.0, "hysteresis": 1.0, "k_max": 4}, "horizon": 600.0})
    assert not any(r["switched"] for r in out["rounds"])
