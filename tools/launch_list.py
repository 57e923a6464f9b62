"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
profiles/: per-kernel mean launch time and share of the serialised total.

    python tools/launch_list.py gpurun_out/launches.csv --cmd "..." --out profiles/r1_launches_v8.json
"""
from __future__ import annotations

import argparse
import collections
import csv
import json
import re


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--cmd", default="")
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    lines = [l for l in open(args.csv) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    launches = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"^essl::", "", r["Kernel Name"].split("(")[0])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "nsecond": 1, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        launches.append({"kernel": name, "ns": ns})
    per = collections.defaultdict(list)
    for l in launches:
        per[l["kernel"]].append(l["ns"])
    tot = sum(sum(v) for v in per.values())
    out = {"cmd": args.cmd,
           "note": "cold-cache, serialised per-launch times; shares, not absolutes, compare with the bench line",
           "mean_ns": {k: sum(v) / len(v) for k, v in per.items()},
           "share": {k: sum(v) / tot for k, v in per.items()},
           "launches": launches}
    with open(args.out, "w") as f:
        json.dump(out, f, indent=0)
    print(json.dumps({"mean_ns": out["mean_ns"], "share": out["share"]}, indent=1))


if __name__ == "__main__":
    main()
