"""pipetune CLI subset: simulate | enumerate | compare | tune | gantt.

    python -m paper_2303_01675_b200.cli simulate --config scenario.json [--plan 1f1b|gpipe|kfkb] [--k K]
                                                 [--b B] [--out DIR] [--format json|text]

The config is a ScenarioConfig JSON (schema_version 1; model / cluster /
traces / policy / horizon; unknown keys rejected by the C++ parser).  All
computation happens in libptk (ptk_scenario_json); this module only moves
JSON around and writes artifacts:
  simulate  -> timeline.json (array of {node, device, stream, start, end}) + summary
  enumerate -> candidates.json          compare -> ranked.json
  tune      -> tuning_log.jsonl (one record per round) + throughput.json
  gantt     -> gantt.svg (one row per device x {compute, send, recv})
Exit codes: 0 ok, 2 config error, 3 infeasible model.
Two runs with the same config produce byte-identical artifacts.
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

from . import pipetune as pt

STREAMS = ("compute", "send", "recv")


def _dump(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":")) + "\n"


def _load(path: str) -> dict:
    try:
        cfg = json.loads(Path(path).read_text())
    except (OSError, json.JSONDecodeError) as e:
        raise pt.PipetuneError("ConfigError", f"cannot read config: {e}")
    if not isinstance(cfg, dict):
        raise pt.PipetuneError("ConfigError", "config must be a JSON object")
    return cfg


def _request(cfg: dict, op: str, **extra) -> dict:
    req = {k: v for k, v in cfg.items() if k in ("schema_version", "model", "cluster", "traces", "policy",
                                                   "horizon", "start", "k_max", "plan")}
    req["op"] = op
    req.update({k: v for k, v in extra.items() if v is not None})
    return req


def cmd_simulate(cfg, args):
    plan = dict(cfg.get("plan", {}))
    if args.plan:
        plan["kind"] = args.plan
    if args.k:
        plan["k"] = args.k
    if args.b:
        plan["micro_batch_size"] = args.b
    res = pt.scenario(_request(cfg, "simulate", plan=plan))["result"]
    timeline = [{"node": n, "device": d, "stream": STREAMS[s], "start": a, "end": b}
                for n, d, s, a, b in res["timeline"]]
    summary = {"pipeline_length_ticks": res["pipeline_length"], "pipeline_length": res["pipeline_length"] / 1e9,
               "bubble_fraction": res["bubble_fraction"], "peak_bytes": res["peak"], "plan": plan}
    return {"timeline.json": timeline, "summary.json": summary}, summary


def cmd_enumerate(cfg, args):
    out = pt.scenario(_request(cfg, "enumerate", k_max=args.k_max))
    table = [{"k": k, "b": b, "M": M, "per_device_peak": peaks} for k, b, M, peaks in out["entries"]]
    return {"candidates.json": table}, table


def cmd_compare(cfg, args):
    out = pt.scenario(_request(cfg, "compare"))
    table = [{"k": k, "b": b, "M": M, "estimated_length": L / 1e9} for k, b, M, L in out["ranked"]]
    return {"ranked.json": table}, table


def cmd_tune(cfg, args):
    out = pt.scenario(_request(cfg, "tune"))
    lines = "".join(_dump({"round_time": r["time"], "chosen": r["chosen"], "switched": r["switched"],
                           "estimates": r["estimates"]}) for r in out["rounds"])
    thr = {"throughput": out["throughput"], "iterations": out["iterations"]}
    return {"tuning_log.jsonl": lines, "throughput.json": thr}, {"rounds": len(out["rounds"]),
                                                                 "throughput": out["throughput"]}


def gantt_svg(res: dict, devices: int) -> str:
    tl = res["timeline"]
    end = max((e[4] for e in tl), default=1) or 1
    W, row = 1000.0, 18
    colors = {0: "#4e79a7", 1: "#f28e2b", 2: "#59a14f"}
    parts = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{int(W) + 120}" height="{devices * 3 * row + 20}">']
    for d in range(devices):
        for s in range(3):
            y = (d * 3 + s) * row + 10
            parts.append(f'<text x="2" y="{y + 12}" font-size="10">dev{d} {STREAMS[s]}</text>')
    for n, d, s, a, b in tl:
        y = (d * 3 + s) * row + 10
        x0, x1 = 110 + W * a / end, 110 + W * b / end
        parts.append(f'<rect x="{x0:.2f}" y="{y}" width="{max(x1 - x0, 0.5):.2f}" height="{row - 3}" '
                     f'fill="{colors[s]}"><title>node {n}</title></rect>')
    parts.append("</svg>\n")
    return "\n".join(parts)


def cmd_gantt(cfg, args):
    files, summary = cmd_simulate(cfg, args)
    res = pt.scenario(_request(cfg, "simulate", plan=summary["plan"]))["result"]
    files["gantt.svg"] = gantt_svg(res, len(cfg["model"]["stages"]))
    return files, summary


COMMANDS = {"simulate": cmd_simulate, "enumerate": cmd_enumerate, "compare": cmd_compare, "tune": cmd_tune,
            "gantt": cmd_gantt}


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="pipetune")
    p.add_argument("command", choices=sorted(COMMANDS))
    p.add_argument("--config", required=True)
    p.add_argument("--out", default="")
    p.add_argument("--format", choices=["json", "text"], default="json")
    p.add_argument("--seed", type=int, default=0, help="reserved: seeded trace generators")
    p.add_argument("--plan", choices=["1f1b", "gpipe", "kfkb"])
    p.add_argument("--k", type=int)
    p.add_argument("--b", type=int)
    p.add_argument("--k-max", type=int)
    args = p.parse_args(argv)
    try:
        cfg = _load(args.config)
        files, summary = COMMANDS[args.command](cfg, args)
    except pt.PipetuneError as e:
        print(f"error: {e}", file=sys.stderr)
        return 3 if e.kind == "InfeasibleModel" else 2
    if args.out:
        out = Path(args.out)
        out.mkdir(parents=True, exist_ok=True)
        for name, content in files.items():
            (out / name).write_text(content if isinstance(content, str) else _dump(content))
    if args.format == "json":
        sys.stdout.write(_dump(summary))
    else:
        for k, v in (summary.items() if isinstance(summary, dict) else enumerate(summary)):
            print(f"{k}: {v}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
