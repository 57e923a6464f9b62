"""Fill / drain view of a tools/timeline.py JSON: running launches per kernel
in 0.1 ms bins, and each batch's span (first launch start -> last end).
    python tools/tl_bins.py gpurun_out/x.json [--bin 0.1]"""
from __future__ import annotations

import argparse
import json


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--bin", type=float, default=0.1)
    a = ap.parse_args()
    d = json.load(open(a.path))
    recs = d["launches"]
    t_end = max(r["end"] for r in recs)
    kinds = sorted({r["kernel"] for r in recs})
    print("summary:", d["summary"]["total_ms"], "ms total;", "kernels", kinds)
    nb = int(t_end / a.bin) + 1
    print("  t(ms) " + " ".join(f"{k[:7]:>7s}" for k in kinds))
    for i in range(nb):
        t0, t1 = i * a.bin, (i + 1) * a.bin
        row = []
        for k in kinds:
            # average number of running launches of kernel k in the bin
            occ = sum(max(0.0, min(t1, r["end"]) - max(t0, r["start"])) for r in recs if r["kernel"] == k) / a.bin
            row.append(occ)
        print(f"  {t0:5.2f} " + " ".join(f"{x:7.2f}" for x in row))
    # batches: per stream, split launches into batches at each 'prep' (or gather)
    spans = []
    for s in sorted({r["stream"] for r in recs}):
        rs = sorted([r for r in recs if r["stream"] == s], key=lambda r: r["start"])
        cur = []
        for r in rs:
            if r["kernel"] in ("prep", "gather") and cur and any(c["kernel"] == r["kernel"] for c in cur):
                spans.append((s, cur[0]["start"], cur[-1]["end"], {c["kernel"]: round(c["end"] - c["start"], 3) for c in cur}))
                cur = []
            cur.append(r)
        if cur:
            spans.append((s, cur[0]["start"], cur[-1]["end"], {c["kernel"]: round(c["end"] - c["start"], 3) for c in cur}))
    for s, a0, a1, ks in sorted(spans, key=lambda x: x[1]):
        print(f"  batch s{s}: {a0:6.3f} -> {a1:6.3f} ({a1 - a0:.3f} ms) {ks}")


if __name__ == "__main__":
    main()
