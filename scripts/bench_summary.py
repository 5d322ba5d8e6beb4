import json,sys
for f in sys.argv[1:]:
    try:
        lines=open(f).read().strip().splitlines()
        d=json.loads(lines[-1])
    except Exception as e:
        print(f, "unparsable", e); continue
    print(f, "lines", len(lines), "value", d["value"], "n", d["n_gpus"], d["config"].get("candidates_kbM"))
    print("  sweep", {k:v["samples_per_s"] for k,v in (d.get("kfkb_sweep") or {}).items()}, "1f1b", d["schedules"]["1f1b"]["samples_per_s"], "ada", d["schedules"]["ada_grouper"]["kb_per_step"][:3], "...")
    print("  decisions", [(x["chosen"], x["switched"]) for x in d["tuner_decisions"]][:12])
    print("  xf", d.get("transfer_forward_ratio",{}) and d["transfer_forward_ratio"]["per_stage"], "hw", d.get("hardware_report",{}).get("length_ratio_measured_over_simulated"), "e2e", d["e2e"]["value"], "clk", d["clocks"])
