"""A/B throughput of two libessl builds on the bench workload, interleaved
runs (device value, longer timed region than the default bench):
    python tools/ab.py --a paper_2404_00509_b200/_lib/libessl.so --b _libB/libessl.so [--n 5]"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--a", required=True)
    ap.add_argument("--b", required=True)
    ap.add_argument("--n", type=int, default=5)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--extra", default="")
    args = ap.parse_args()
    res = {"a": [], "b": []}
    for i in range(args.n):
        for k in ("a", "b"):
            env = dict(os.environ, ESSL_LIB=str(Path(getattr(args, k)).resolve()))
            cmd = [sys.executable, str(ROOT / "bench.py"), "--no-cpu", "--no-e2e", "--steps",
                   str(args.steps)] + args.extra.split()
            r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)
            try:
                v = json.loads(r.stdout.strip().splitlines()[-1])["value"]
            except Exception:
                print(k, "failed", r.stderr[-500:], file=sys.stderr)
                continue
            res[k].append(v)
            print(k, round(v), flush=True)
    out = {k: {"median": round(statistics.median(v)), "runs": [round(x) for x in v]} for k, v in res.items() if v}
    if res["a"] and res["b"]:
        out["b_over_a"] = round(statistics.median(res["b"]) / statistics.median(res["a"]), 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
