"""CLI subset: artifacts, exit codes 0/2/3, byte-identical reruns (acceptance 9)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2303_01675_b200 import cli  # noqa: E402

FIG2 = str(ROOT / "examples" / "fig2_scenario.json")
TWO = str(ROOT / "examples" / "two_regime_scenario.json")


def test_simulate_artifacts_and_determinism(tmp_path):
    for run in ("a", "b"):
        assert cli.main(["gantt", "--config", FIG2, "--out", str(tmp_path / run)]) == 0
    for name in ("timeline.json", "summary.json", "gantt.svg"):
        assert (tmp_path / "a" / name).read_bytes() == (tmp_path / "b" / name).read_bytes()
    tl = json.loads((tmp_path / "a" / "timeline.json").read_text())
    assert {"node", "device", "stream", "start", "end"} <= set(tl[0])


def test_tune_log_is_jsonl_and_deterministic(tmp_path):
    for run in ("a", "b"):
        assert cli.main(["tune", "--config", TWO, "--out", str(tmp_path / run)]) == 0
    a = (tmp_path / "a" / "tuning_log.jsonl").read_bytes()
    assert a == (tmp_path / "b" / "tuning_log.jsonl").read_bytes()
    rounds = [json.loads(x) for x in a.decode().splitlines()]
    assert any(r["switched"] for r in rounds)


def test_exit_codes(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"model": {"global_batch": 4, "stages": [{}]}, "plan": {"micro_batch_size": 3}}))
    assert cli.main(["simulate", "--config", str(bad)]) == 2       # b does not divide global batch
    unk = tmp_path / "unk.json"
    unk.write_text(json.dumps({"model": {"global_batch": 4, "stages": [{"bogus": 1}]}}))
    assert cli.main(["simulate", "--config", str(unk)]) == 2       # unknown key rejected
    inf = tmp_path / "inf.json"
    inf.write_text(json.dumps({"model": {"global_batch": 4, "stages": [{"weight_bytes": 1000}]},
                               "cluster": {"device_memory_limit": 10, "devices": 1}}))
    assert cli.main(["enumerate", "--config", str(inf)]) == 3      # InfeasibleModel


def test_missing_required_fields_are_config_errors(tmp_path):
    """Mandatory request fields missing -> ConfigError / exit code 2, never a crash
    (enumerate without a cluster, tune without a horizon, simulate without a plan)."""
    model = {"global_batch": 4, "stages": [{}, {}]}
    cases = [("enumerate", {"model": model}),
             ("tune", {"model": model, "cluster": {"device_memory_limit": 10**12, "devices": 2},
                       "traces": [{"link": 0}, {"link": 1}]}),
             ("compare", {"model": model})]
    for cmd, cfg in cases:
        p = tmp_path / f"{cmd}.json"
        p.write_text(json.dumps(cfg))
        assert cli.main([cmd, "--config", str(p)]) == 2, cmd


def test_abi_missing_keys_return_config_error():
    from paper_2303_01675_b200 import pipetune as pt
    import pytest
    model = {"global_batch": 4, "stages": [{}]}
    for req in ({"op": "decide", "model": model}, {"op": "transfer"}, {"op": "estimate", "samples": []},
                {"op": "simulate", "model": model}, {"op": "decide", "model": model, "candidates": [[1]],
                                                    "compute_profile": [], "samples": []}):
        with pytest.raises(pt.PipetuneError) as e:
            pt.scenario(req)
        assert e.value.kind == "ConfigError", (req, e.value.kind)
