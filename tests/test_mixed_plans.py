"""Mixed-k (group-list) candidates in the Ada-Grouper decision (reference
make_plan walks any group list, plan.cpp:20-21, 61-66).

Under the constant profiled durations the cost model is defined on, a mixed plan
pays off when k does not divide M: putting the remainder group FIRST shortens the warm-up that
uniform kFkB's short LAST group does not.  The C++ decision (scenario op "decide" with
group_candidates) must equal the oracle bit for bit, and must pick the remainder-first plan in
that case (a switch from the uniform incumbent, reported with chosen_groups)."""
import copy
import random

import pytest

from oracle import spec_oracle as O
from paper_2303_01675_b200 import pipetune as pt


def _request(S, gb, cands, mixed, f_ns, b_ns, x_ns, out_bytes=100, current=None, current_groups=None):
    model = {"global_batch": gb, "stages": [{"output_bytes_per_sample_fwd": out_bytes,
                                              "output_bytes_per_sample_bwd": out_bytes} for _ in range(S)]}
    bs = sorted({c[1] for c in cands} | {m[0] for m in mixed})
    comp = [[s, b, d, (f_ns if d == 0 else b_ns) * b] for s in range(S) for b in bs for d in (0, 1)]
    samples = [[l, b * out_bytes, 0, x_ns * b] for l in range(2 * (S - 1)) for b in bs for _ in range(3)]
    req = {"op": "decide", "model": model, "candidates": cands, "group_candidates": mixed, "compute_profile": comp,
           "samples": samples, "hysteresis": 0.02, "window": 8, "clock": 7}
    if current is not None:
        req["current"] = current
    if current_groups is not None:
        req["current_groups"] = current_groups
    return req


def test_remainder_first_beats_uniform_when_k_does_not_divide_m():
    S, M = 4, 10
    req = _request(S, M, [[k, 1, M] for k in (1, 2, 4)], [[1, [2, 4, 4]], [1, [1, 1, 4, 4]]],
                   1_000_000, 2_000_000, 1_500_000, current=[4, 1, M])
    got = pt.scenario(req)["decision"]
    assert got == O.run(copy.deepcopy(req))["decision"]
    assert got["switched"] and got["chosen"][0] == 4 and got["chosen_groups"] in ([2, 4, 4], [1, 1, 4, 4])
    uniform4 = [e for e in got["estimates"] if e[:3] == [4, 1, M] and len(e) == 4][0]
    assert got["estimates"][0][3] < uniform4[3]


def test_mixed_incumbent_and_unknown_groups():
    S, M = 2, 8
    req = _request(S, M, [[k, 1, M] for k in (1, 2)], [[1, [1, 2, 2, 3]]], 1_000_000, 2_000_000, 500_000,
                   current=[3, 1, M], current_groups=[1, 2, 2, 3])
    assert pt.scenario(req)["decision"] == O.run(copy.deepcopy(req))["decision"]
    req["current_groups"] = [3, 3, 2]
    with pytest.raises(pt.PipetuneError) as e:
        pt.scenario(req)
    assert e.value.kind == "UnknownCandidate"


@pytest.mark.parametrize("seed", range(40))
def test_decide_with_group_candidates_matches_oracle(seed):
    rng = random.Random(seed)
    S = rng.randint(2, 5)
    M = rng.choice([6, 8, 9, 10, 12, 16])
    ks = sorted({rng.randint(1, M) for _ in range(3)})
    mixed = []
    for _ in range(rng.randint(1, 4)):
        sizes, left = [], M
        while left:
            n = rng.randint(1, min(left, 5))
            sizes.append(n)
            left -= n
        mixed.append([1, sizes])
    req = _request(S, M, [[k, 1, M] for k in ks], mixed, rng.choice([500_000, 1_000_000]),
                   rng.choice([1_000_000, 2_000_000]), rng.choice([0, 300_000, 1_500_000]))
    if rng.random() < 0.5:
        req["current"] = [ks[0], 1, M]
    assert pt.scenario(req)["decision"] == O.run(copy.deepcopy(req))["decision"]
