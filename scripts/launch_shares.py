"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv`) into per-kernel
launch counts, summed device time and share, as a markdown table (profiles/*.md).

    python scripts/launch_shares.py gpurun_out/launches.csv [--top 20]
"""
import argparse
import csv
import re
from collections import defaultdict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=20)
    a = ap.parse_args()
    with open(a.csv) as f:
        rows = [ln for ln in f if ln.startswith('"')]
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in csv.DictReader(rows):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"^void ", "", r["Kernel Name"])
        name = re.sub(r"\(.*$", "", re.sub(r"^\(?anonymous namespace\)::|^unnamed>::", "", name))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
        tot[name] += float(r["Metric Value"].replace(",", "")) * scale
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{sum(cnt.values())} launches, {s / 1e3:.1f} ms serialised device time\n")
    print("| kernel | launches | total µs | share |\n|---|---|---|---|")
    for k in sorted(tot, key=tot.get, reverse=True)[: a.top]:
        print(f"| {k} | {cnt[k]} | {tot[k]:.1f} | {100 * tot[k] / s:.1f}% |")


if __name__ == "__main__":
    main()
