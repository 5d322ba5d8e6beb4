"""bubble_report / queue_analysis of a measured pipeline iteration (SPEC.md:351-361 on hardware).

Every stage's executor timeline (ptk_exec_timeline_json: compute and transfer records in ns from
its iteration start, plus that start on the GPU's %globaltimer) is put on one clock and handed to
the C++ `result_from_records` (scenario op "hardware_report"), which applies the simulator's own
definitions: busy, bubble = active span - busy, and for every launch with an input whether that
input had landed before the device was free.  Beside it, the cost model's prediction for the same
plan (op "estimate_sim": simulate over constant durations) fed the run's own mean
forward / backward / transfer times — the GPU-vs-simulate() diff.  GradAccum records are left out:
the simulator gives GradAccum zero duration.
"""
from __future__ import annotations

import statistics

from . import pipetune as pt


def _plan(tl: dict) -> dict:
    return {"kind": "groups", "groups": list(tl["groups"]), "micro_batch_size": int(tl["b"])}


def pipeline_report(timelines: list[dict], model: dict, clock_offsets_ns: list[int] | None = None) -> dict:
    """timelines[s] = stage s's timeline dict; model = the pipetune ModelSpec dict the executor's
    graph was built from (tuning.pipeline_model); clock_offsets_ns[s] = stage s's globaltimer minus
    stage 0's at a common instant (0 on one GPU)."""
    S = len(timelines)
    offs = clock_offsets_ns or [0] * S
    t0 = [int(tl["t0_globaltimer"]) - int(o) for tl, o in zip(timelines, offs)]
    base = min(t0)
    comp, xfer = [], []
    fwd = [[] for _ in range(S)]
    bwd = [[] for _ in range(S)]
    samples = []
    for s, tl in enumerate(timelines):
        d = t0[s] - base
        for node, kind, mb, start, end in tl["compute"]:
            if kind == 2:
                continue  # GradAccum: zero duration in the simulator
            comp.append([s, int(node), d + int(start), d + int(end)])
            (fwd if kind == 0 else bwd)[s].append(int(end) - int(start))
        for link, mb, nbytes, start, end in tl["xfer"]:
            xfer.append([int(link), int(mb), d + int(start), d + int(end)])
            samples.append([int(link), int(nbytes), 0, int(end) - int(start)])
    plan = _plan(timelines[0])
    hw = pt.scenario({"op": "hardware_report", "model": model, "plan": plan,
                      "records": {"compute": comp, "xfer": xfer}, "start": 0})["result"]
    b = plan["micro_batch_size"]
    prof = []
    for s in range(S):
        prof.append([s, b, 0, int(statistics.mean(fwd[s]))])
        prof.append([s, b, 1, int(statistics.mean(bwd[s]))])
    sim = pt.scenario({"op": "estimate_sim", "model": model, "plan": plan, "compute_profile": prof,
                       "samples": samples, "window": max(1, len(samples))})["result"]

    def summary(r):
        launches = [x for d in r["launches"] for x in d]
        return {"pipeline_length_ns": r["pipeline_length"],
                "bubble_fraction": [round(x, 4) for x in r["bubble_fraction"]],
                "prebuffered_launches": sum(1 for x in launches if x[1]), "launches_with_input": len(launches)}

    m, p = summary(hw), summary(sim)
    return {"measured": m, "simulated": p,
            "length_ratio_measured_over_simulated": round(m["pipeline_length_ns"] / max(1, p["pipeline_length_ns"]), 4),
            "queue_analysis": [[x[1] for x in d] for d in hw["launches"]],
            "inputs": {"fwd_ns": [row[3] for row in prof[0::2]], "bwd_ns": [row[3] for row in prof[1::2]]}}
