"""Generate tests/golden/planner_ref.json from the COMPILED REFERENCE planner.

Runs oracle/_ref/ref_dump (built by `make -C oracle` from the unmodified
/root/reference/proj/src sources) over the parity grid and stores, per case,
the sha256 of its canonical JSON dump, plus the full dump of a few small
cases.  The GPU box has no /root/reference; tests there use this file.

    make -C oracle && python tests/golden/make_planner_golden.py
"""
import hashlib
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
REF = ROOT / "oracle" / "_ref" / "ref_dump"
OUT = Path(__file__).with_name("planner_ref.json")
C1 = Path(__file__).with_name("c1_sequences.json")


def grid():
    cases = []
    for S in range(1, 7):
        for M in range(1, 13):
            for b in (1, 2):
                cases.append((S, M, b, 0, 1))
                cases.append((S, M, b, 2, 1))
                for k in range(0, M + 2):  # includes k=0 and k=M+1 (PlanError)
                    cases.append((S, M, b, 1, k))
    for S, M, ks in ((8, 32, (1, 2, 3, 4, 8, 32)), (8, 64, (1, 4, 6)), (4, 16, (1, 2, 3, 4)), (7, 20, (3,))):
        for k in ks:
            cases.append((S, M, 2, 1, k))
    return cases


def run(cases, fwd=10, bwd=7):
    inp = "".join(f"{S} {M} {b} {kind} {k} {fwd} {bwd}\n" for S, M, b, kind, k in cases)
    r = subprocess.run([str(REF)], input=inp, capture_output=True, text=True, check=True)
    return r.stdout.splitlines()


def main():
    cases = grid()
    lines = run(cases)
    assert len(lines) == len(cases)
    small = {(2, 4, 1, 0, 1), (2, 4, 1, 1, 2), (1, 2, 1, 0, 1), (2, 2, 1, 2, 1), (4, 16, 2, 1, 3)}
    out = {"generator": "oracle/_ref/ref_dump (reference proj/src/{model,taskgraph,plan}.cpp, g++ -O2)",
           "payload": {"fwd_base": 10, "bwd_base": 7}, "cases": []}
    for c, line in zip(cases, lines):
        e = {"case": list(c), "sha256": hashlib.sha256(line.encode()).hexdigest()}
        if c in small:
            e["json"] = json.loads(line)
        out["cases"].append(e)
    OUT.write_text(json.dumps(out, separators=(",", ":")) + "\n")
    print(f"wrote {len(cases)} cases to {OUT}")
    # configs[0] (C1 toy: S=4, M=16, b=1) per-device sequences for k = 1, 2, 4, 16 (GPipe-equivalent):
    # what the GPU executor's recorded order must equal (tests/test_pipeline_gpu.py)
    c1 = [(4, 16, 1, 1, k) for k in (1, 2, 4, 16)] + [(2, 8, 1, 1, k) for k in (1, 2, 4)]
    seqs = {f"S{S}_M{M}_b{b}_k{k}": json.loads(line)["sequences"] for (S, M, b, _, k), line in zip(c1, run(c1))}
    C1.write_text(json.dumps({"generator": out["generator"], "sequences": seqs}, indent=1) + "\n")
    print(f"wrote {len(seqs)} C1 sequence sets to {C1}")


if __name__ == "__main__":
    sys.exit(main())
