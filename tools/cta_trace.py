"""Per-CTA execution trace of the pipelined loader (ESSL_OPT_TRACE): how the
CTAs of k_prep / k_entropy / k_idct / k_resize share the SMs over time.

    python tools/cta_trace.py [--streams 6] [--steps 40] [--out profiles/x.json]

Prints, over the traced window: mean resident CTAs per SM by kernel, SM-time
with no traced CTA, CTA durations, and entropy CTAs' duration vs how many
other CTAs shared their SM."""

from __future__ import annotations

import argparse
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
NAMES = {6: "prep", 7: "entropy", 8: "idct", 1: "resize"}


def main():
    import torch
    import paper_2404_00509_b200 as E
    from paper_2404_00509_b200 import _native as N, build
    build.build()
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=6)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--pool", type=int, default=4096)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    path = Path(tempfile.mkdtemp()) / "pool.essl"
    E.build_synthetic(path, args.pool, 256, 95, classes=1000, seed=1)
    cfg = E.LoaderConfig(data=str(path), batch_size=256, res=224, out_dtype="bfloat16",
                         mask_ratio=0.75, streams=args.streams, prefetch=args.streams,
                         reuse_outputs=True)
    loader = E.Loader(cfg)
    perm = E.epoch_permutation(0, 0, len(loader.handle))
    nb = len(perm) // 256
    pend = []
    for i in range(30):
        pend.append(loader.enqueue(0, perm[(i % nb) * 256:][:256]))
        if len(pend) > 2 * args.streams:
            loader.finish(pend.pop(0))
    for p in pend:
        loader.finish(p)
    cap = 1 << 20
    for e in loader.engines:
        e.set_option(N.ESSL_OPT_TRACE, cap)
    torch.cuda.synchronize()
    pend = []
    for i in range(args.steps):
        pend.append(loader.enqueue(0, perm[(i % nb) * 256:][:256]))
        if len(pend) > 2 * args.streams:
            loader.finish(pend.pop(0))
    for p in pend:
        loader.finish(p)
    recs = []
    for e in loader.engines:
        buf = np.zeros((cap, 4), np.uint64)
        n = N.lib().essl_trace_read(e._ctx, N.ptr(buf), cap)
        N.check(min(n, 0), "essl_trace_read")
        recs.append(buf[:n])
        e.set_option(N.ESSL_OPT_TRACE, 0)
    r = np.concatenate(recs).astype(np.int64)
    t0 = r[:, 0].min()
    r[:, 0] -= t0
    r[:, 1] -= t0
    # steady-state window: the middle of the longest stretch with entropy CTAs
    # resident throughout (host stalls leave gaps in the trace)
    e = r[r[:, 2] == 7]
    ev = sorted([(a, 1) for a in e[:, 0]] + [(b, -1) for b in e[:, 1]])
    runs, cur, start = [], 0, None
    for t, dlt in ev:
        if cur == 0 and dlt > 0:
            start = t
        cur += dlt
        if cur == 0 and start is not None:
            runs.append((start, t))
            start = None
    a0, b0 = max(runs, key=lambda ab: ab[1] - ab[0])
    lo, hi = int(a0 + 0.1 * (b0 - a0)), int(b0 - 0.1 * (b0 - a0))
    win = hi - lo
    nsm = int(r[:, 3].max()) + 1
    out = {"window_us": win / 1e3, "sms": nsm, "ctas": int(len(r))}
    occ = {}
    for kid, name in NAMES.items():
        m = r[:, 2] == kid
        a = np.clip(r[m, 0], lo, hi)
        b = np.clip(r[m, 1], lo, hi)
        occ[name] = float((b - a).sum()) / (win * nsm)
        d = (r[m, 1] - r[m, 0]) / 1e3
        out[f"{name}_cta_us"] = {"median": round(float(np.median(d)), 1),
                                 "p90": round(float(np.percentile(d, 90)), 1), "n": int(m.sum())}
    out["mean_resident_ctas_per_sm"] = {k: round(v, 2) for k, v in occ.items()}
    # SM idle (no traced CTA) fraction in the window
    idle = 0
    for sm in range(nsm):
        m = r[:, 3] == sm
        iv = sorted(zip(np.clip(r[m, 0], lo, hi), np.clip(r[m, 1], lo, hi)))
        cur, busy = lo, 0
        for a, b in iv:
            if b <= cur:
                continue
            busy += b - max(a, cur)
            cur = max(cur, b)
        idle += win - busy
    out["sm_idle_frac"] = round(idle / (win * nsm), 4)
    m = (r[:, 2] == 7) & (r[:, 1] >= lo) & (r[:, 1] < hi)
    out["img_per_s_in_window"] = round(float(m.sum()) / (win / 1e9))
    warps = {"prep": 8, "entropy": 2, "idct": 8, "resize": 8}
    out["mean_resident_warps_per_sm"] = round(sum(occ[k] * warps[k] for k in occ), 1)
    print(json.dumps(out, indent=1))
    if args.out:
        Path(args.out).write_text(json.dumps({"summary": out, "records": r.tolist()}))


if __name__ == "__main__":
    main()
