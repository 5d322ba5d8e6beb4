"""bubble_report / queue_analysis on measured timelines (§8(a) a17).

`result_from_records` (C++, op "hardware_report") turns the executor's per-stage compute and
transfer records into a SimResult.  Its pin: fed the simulator's own timeline (random scenarios,
SPEC-faithful traces) it must reproduce simulate()'s busy / bubble / pre-buffered launches / queue
depth / pipeline length exactly — so on the GPU the same definitions are applied to real timestamps.
"""
import random

import pytest

from paper_2303_01675_b200 import pipetune as pt
from tests.spec_scenarios import random_scenario

KINDS = {"1f1b": pt.PLAN_1F1B, "kfkb": pt.PLAN_KFKB, "gpipe": pt.PLAN_GPIPE}


def records_from_sim(req, res):
    model = pt.ModelSpec([pt.StageProfile(stage_id=i, **st) for i, st in enumerate(req["model"]["stages"])],
                         req["model"]["global_batch"])
    p = req["plan"]
    plan = pt.plan(model, p["micro_batch_size"], KINDS[p["kind"]], p.get("k", 1))
    comp, xfer = [], []
    for node, dev, stream, start, end in res["timeline"]:
        if stream == 0:
            comp.append([dev, node, start, end])
        elif stream == 1:
            kind, stage, mb, device, link, payload = plan["nodes"][node]
            xfer.append([link, mb, start, end])
    return {"compute": comp, "xfer": xfer}


@pytest.mark.parametrize("seed", range(120))
def test_records_of_simulation_reproduce_simulate(seed):
    rng = random.Random(seed)
    req = random_scenario(rng)
    res = pt.scenario(req)["result"]
    hw = pt.scenario({"op": "hardware_report", "model": req["model"], "plan": req["plan"],
                      "records": records_from_sim(req, res), "start": req["start"]})["result"]
    for key in ("pipeline_length", "busy", "bubble", "bubble_fraction", "launches"):
        assert hw[key] == res[key], key
    assert [sorted(d) for d in hw["queue_depth"]] == [sorted(d) for d in res["queue_depth"]]


def test_records_outside_the_plan_are_config_errors():
    req = random_scenario(random.Random(3))
    while len(req["model"]["stages"]) < 2:
        req = random_scenario(random.Random(req["start"] + 7))
    bad = {"compute": [[0, 10**6, 0, 1]], "xfer": []}
    with pytest.raises(pt.PipetuneError) as e:
        pt.scenario({"op": "hardware_report", "model": req["model"], "plan": req["plan"], "records": bad})
    assert e.value.kind == "ConfigError"
