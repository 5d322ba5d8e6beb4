"""Planner parity: libptk's C++ planner vs the COMPILED REFERENCE planner.

The reference (proj/src/{model,taskgraph,plan}.cpp) is compiled unmodified by
oracle/Makefile into oracle/_ref/ref_dump; tests/golden/planner_ref.json holds
the sha256 of its JSON dump for 1526 cases (S<=6, M<=12, every k incl. the
out-of-range k=0 and k=M+1, b in {1,2}, plus S=8 M=32/64 cases).  Our dump
(ptk_plan_json) must match byte for byte: node ids, edges, lookup tables,
per-device orders, units, sequences, validate(), check_plan(), topo order.
"""
import hashlib
import json
import shutil
import subprocess
from pathlib import Path

import pytest

from paper_2303_01675_b200 import pipetune as pt

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = json.loads((ROOT / "tests" / "golden" / "planner_ref.json").read_text())
REF_BIN = ROOT / "oracle" / "_ref" / "ref_dump"


def _mine(case):
    S, M, b, kind, k = case
    model = pt.uniform_model(S, M * b, GOLDEN["payload"]["fwd_base"], GOLDEN["payload"]["bwd_base"])
    return pt.plan_json_str(model, b, kind, k)


def test_golden_grid_bit_exact():
    bad = []
    for e in GOLDEN["cases"]:
        s = _mine(tuple(e["case"]))
        if hashlib.sha256(s.encode()).hexdigest() != e["sha256"]:
            bad.append(e["case"])
    assert not bad, f"{len(bad)} cases differ from the reference, first: {bad[:5]}"


def test_golden_full_dumps():
    for e in GOLDEN["cases"]:
        if "json" in e:
            assert json.loads(_mine(tuple(e["case"]))) == e["json"]


@pytest.mark.skipif(not REF_BIN.exists(), reason="reference oracle not built (make -C oracle)")
def test_live_reference_random_payloads():
    """Different payload bases than the golden grid, straight against the live reference binary."""
    cases = [(S, M, b, 1, k) for S in (1, 3, 5) for M in (1, 5, 9) for b in (1, 3) for k in (1, 2, M)]
    inp = "".join(f"{S} {M} {b} {kind} {k} 123 45\n" for S, M, b, kind, k in cases)
    ref = subprocess.run([str(REF_BIN)], input=inp, capture_output=True, text=True, check=True).stdout.splitlines()
    for c, r in zip(cases, ref):
        S, M, b, kind, k = c
        mine = pt.plan_json_str(pt.uniform_model(S, M * b, 123, 45), b, kind, k)
        assert mine == r, c


# ---- SPEC.md examples (Appendix A of SURVEY.md), asserted directly ----------------------------

def _seqs(S, M, kind, k=1):
    p = pt.plan(pt.uniform_model(S, M), 1, kind, k)
    return [s.replace(" GA", "").replace("GA", "") for s in p["sequences"]]


def test_spec_planner_examples():
    assert _seqs(2, 4, pt.PLAN_1F1B) == ["F0 F1 B0 F2 B1 F3 B2 B3", "F0 B0 F1 B1 F2 B2 F3 B3"]
    assert _seqs(2, 4, pt.PLAN_KFKB, 2) == ["F0 F1 F2 F3 B0 B1 B2 B3", "F0 F1 B0 B1 F2 F3 B2 B3"]
    assert _seqs(1, 2, pt.PLAN_1F1B) == ["F0 B0 F1 B1"]
    assert _seqs(2, 2, pt.PLAN_GPIPE)[0] == "F0 F1 B0 B1"
    assert _seqs(1, 3, pt.PLAN_GPIPE) == ["F0 F1 F2 B0 B1 B2"]


def test_graph_counts_closed_form():
    # M*S F, M*S B, 2M(S-1) Send, 2M(S-1) Recv, S GA; edges M(7S-5)
    for S in range(1, 9):
        for M in range(1, 17):
            p = pt.plan(pt.uniform_model(S, M), 1, pt.PLAN_1F1B)
            kinds = [n[0] for n in p["nodes"]]
            assert [kinds.count(i) for i in range(5)] == [M * S, M * S, 2 * M * (S - 1), 2 * M * (S - 1), S]
            assert len(p["edges"]) == M * (7 * S - 5)
            assert p["violations"] == [] and p["check"] == 0


def test_plan_identities_and_ascending_order():
    # SPEC.md:181 identities, and the ascending-micro-batch property the GPU relies on
    for S in range(1, 7):
        for M in range(1, 13):
            m = pt.uniform_model(S, M)
            one = pt.plan(m, 1, pt.PLAN_1F1B)
            gp = pt.plan(m, 1, pt.PLAN_GPIPE)
            for k in range(1, M + 1):
                p = pt.plan(m, 1, pt.PLAN_KFKB, k)
                assert p["check"] == 0
                if k == 1:
                    assert p["per_device"] == one["per_device"]
                if k == M:
                    assert p["per_device"] == gp["per_device"]
                for seq in p["sequences"]:
                    toks = seq.split()
                    f = [int(t[1:]) for t in toks if t[0] == "F"]
                    b = [int(t[1:]) for t in toks if t[0] == "B"]
                    assert f == sorted(f) and b == sorted(b)


def test_errors_are_typed():
    with pytest.raises(pt.PipetuneError) as e:
        pt.plan_kfkb(pt.uniform_model(2, 4), 1, 5)
    assert e.value.kind == "PlanError"
    with pytest.raises(pt.PipetuneError) as e:
        pt.plan_kfkb(pt.uniform_model(2, 4), 3, 1)  # b=3 does not divide 4
    assert e.value.kind == "ConfigError"


def test_reference_harness_source_compatible_with_our_headers(tmp_path):
    """Drop-in at the C++ source level: the SAME harness source that links the reference planner
    (oracle/ref_dump.cpp) compiles against OUR include/pipetune headers, links libptk.so instead of
    the reference objects, and prints byte-identical output over the whole golden grid."""
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    from paper_2303_01675_b200 import _lib as L
    exe = tmp_path / "ref_dump_ptk"
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "oracle" / "ref_dump.cpp"),
                    f"-L{L.LIB_PATH.parent}", "-lptk", f"-Wl,-rpath,{L.LIB_PATH.parent}", "-o", str(exe)],
                   check=True, capture_output=True)
    fwd, bwd = GOLDEN["payload"]["fwd_base"], GOLDEN["payload"]["bwd_base"]
    inp = "".join(f"{S} {M} {b} {kind} {k} {fwd} {bwd}\n" for S, M, b, kind, k in (e["case"] for e in GOLDEN["cases"]))
    out = subprocess.run([str(exe)], input=inp, capture_output=True, text=True, check=True).stdout.splitlines()
    assert len(out) == len(GOLDEN["cases"])
    bad = [e["case"] for e, line in zip(GOLDEN["cases"], out)
           if hashlib.sha256(line.encode()).hexdigest() != e["sha256"]]
    assert not bad, bad[:5]
