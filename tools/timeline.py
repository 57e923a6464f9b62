"""Per-launch GPU timeline of the loader (CUDA events around every libessl
launch, relative to one reference event): where the batches overlap.

    python tools/timeline.py [--streams 3] [--steps 40] [--out profiles/x.json]
"""

from __future__ import annotations

import argparse
import json
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=3)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--pool", type=int, default=4096)
    ap.add_argument("--out", default=None)
    ap.add_argument("--host", action="store_true", help="pinned-container bus gather (resident=False)")
    ap.add_argument("--gather-ctas", type=int, default=-1, help="ESSL_OPT_GATHER_CTAS (-1: default)")
    ap.add_argument("--staging", default="gather", choices=["gather", "copy"])
    ap.add_argument("--gather-tma", type=int, default=-1)
    args = ap.parse_args()
    import ctypes

    import numpy as np
    import torch

    import paper_2404_00509_b200 as E
    from paper_2404_00509_b200 import _native as N
    d = Path(tempfile.mkdtemp())
    path = d / "pool.essl"
    E.build_synthetic(path, args.pool, 256, 95, seed=3)
    cfg = E.LoaderConfig(data=str(path), batch_size=256, res=224, out_dtype="bfloat16",
                         mask_ratio=0.75, resident=not args.host, streams=args.streams,
                         staging=args.staging,
                         prefetch=args.streams,
                         reuse_outputs=True)
    loader = E.Loader(cfg)
    if args.gather_ctas >= 0:
        loader.set_option(N.ESSL_OPT_GATHER_CTAS, args.gather_ctas)
    if args.gather_tma >= 0:
        loader.set_option(N.ESSL_OPT_GATHER_TMA, args.gather_tma)
    perm = E.epoch_permutation(0, 0, len(loader.handle))
    nb = len(perm) // 256

    def idx(i):
        j = i % nb
        return perm[j * 256:(j + 1) * 256]

    pend = []
    ring_depth = 2 * max(cfg.prefetch, cfg.streams) + 2
    for i in range(max(args.warmup, args.streams * (ring_depth + 1))):
        pend.append(loader.enqueue(0, idx(i)))
        if len(pend) > 2 * args.streams:
            loader.finish(pend.pop(0))
    for p in pend:
        loader.finish(p)
    import gc
    gc.collect()
    gc.freeze()
    torch.cuda.synchronize()
    loader.set_option(N.ESSL_OPT_PROFILE, 1)
    loader.profile_read()
    st = torch.cuda.current_stream()
    N.lib().essl_profile_mark(ctypes.c_void_p(st.cuda_stream))
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(st)
    import time
    pend = []
    host_enq, host_fin = [], []
    for i in range(args.steps):
        h0 = time.perf_counter()
        pend.append(loader.enqueue(0, idx(args.warmup + i)))
        h1 = time.perf_counter()
        if len(pend) > 2 * args.streams:
            loader.finish(pend.pop(0))
        host_enq.append(h1 - h0)
        host_fin.append(time.perf_counter() - h1)
    for p in pend:
        loader.join(p)
    t1.record(st)
    torch.cuda.synchronize()
    total = t0.elapsed_time(t1)
    recs = []
    for s, eng in enumerate(loader.engines):
        for k, a, b in eng.profile_timeline():
            recs.append({"stream": s, "kernel": k, "start": a, "end": b})
    loader.profile_read()
    recs.sort(key=lambda r: r["start"])
    # busy fraction per kernel and GPU-wide "any kernel running"
    ev = sorted([(r["start"], 1) for r in recs] + [(r["end"], -1) for r in recs])
    busy = 0.0
    run = 0
    last = 0.0
    conc = {}
    for t, dlt in ev:
        if run > 0:
            busy += t - last
        conc[run] = conc.get(run, 0.0) + (t - last)
        run += dlt
        last = t
    per = {}
    for r in recs:
        per.setdefault(r["kernel"], []).append(r["end"] - r["start"])
    summ = {"streams": args.streams, "steps": args.steps, "host": args.host,
            "gather_ctas": args.gather_ctas, "gather_tma": args.gather_tma, "staging": args.staging, "total_ms": total,
            "ms_per_step": total / args.steps, "gpu_busy_frac": busy / total,
            "concurrency_ms": {k: round(v, 3) for k, v in sorted(conc.items())},
            "kernel_mean_ms": {k: round(float(np.mean(v)), 4) for k, v in per.items()},
            "host_enqueue_ms": round(1e3 * float(np.median(host_enq)), 3),
            "host_finish_ms": round(1e3 * float(np.median(host_fin)), 3)}
    print(json.dumps(summ))
    # gaps between consecutive launches on each stream
    for s in range(args.streams):
        rs = [r for r in recs if r["stream"] == s]
        gaps = [rs[i + 1]["start"] - rs[i]["end"] for i in range(len(rs) - 1)]
        print(f"stream {s}: launches {len(rs)}, gap mean {np.mean(gaps):.3f} ms, max {np.max(gaps):.3f} ms")
    # gaps by transition (previous kernel -> next kernel on the same stream)
    trans = {}
    for st_ in range(args.streams):
        rs = [r for r in recs if r["stream"] == st_]
        for i in range(len(rs) - 1):
            key = rs[i]["kernel"] + "->" + rs[i + 1]["kernel"]
            trans.setdefault(key, []).append(rs[i + 1]["start"] - rs[i]["end"])
    print("gaps by transition (ms):", {k: (round(float(np.mean(v)), 4), round(float(np.max(v)), 4), len(v))
                                       for k, v in trans.items()})
    mid = len(recs) // 2
    for r in recs[mid:mid + 50]:
        print(f"  s{r['stream']} {r['kernel']:8s} {r['start']:8.3f} {r['end']:8.3f} ({r['end'] - r['start']:.3f})")
    if args.out:
        Path(args.out).write_text(json.dumps({"summary": summ, "launches": recs}, indent=0))


if __name__ == "__main__":
    main()
