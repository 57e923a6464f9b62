"""Interleaved throughput comparison of several libessl builds (each with
optional extra bench args), device value and e2e:
    python tools/abn.py _libA/libessl.so "_libV3/libessl.so|--seq-bits 2048" --n 3"""
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
    ap.add_argument("specs", nargs="+", help="lib[|extra bench args]")
    ap.add_argument("--n", type=int, default=3)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--e2e", action="store_true")
    args = ap.parse_args()
    res = {s: [] for s in args.specs}
    for _ in range(args.n):
        for spec in args.specs:
            lib, _, extra = spec.partition("|")
            env = dict(os.environ, ESSL_LIB=str(Path(lib).resolve()))
            cmd = [sys.executable, str(ROOT / "bench.py"), "--no-cpu", "--steps", str(args.steps)]
            if not args.e2e:
                cmd.append("--no-e2e")
            r = subprocess.run(cmd + extra.split(), capture_output=True, text=True, env=env, timeout=900)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])
            except Exception:
                print(spec, "failed", r.stderr[-400:], file=sys.stderr)
                continue
            res[spec].append((d["value"], (d.get("e2e") or {}).get("value")))
            print(spec, round(d["value"]), flush=True)
    base = None
    for spec, v in res.items():
        if not v:
            continue
        med = statistics.median(x[0] for x in v)
        base = base or med
        e2e = [x[1] for x in v if x[1]]
        print(json.dumps({"spec": spec, "median": round(med), "vs_first": round(med / base, 4),
                          "runs": [round(x[0]) for x in v],
                          "e2e_median": round(statistics.median(e2e)) if e2e else None}))


if __name__ == "__main__":
    main()
