"""Kernel timeline of the bench's e2e leg (Loader.epochs over the page-locked
host container, launch groups as bench.py) for a short timed region: where
the fill and the drain go.  Analysis tool:
    python tools/e2e_timeline.py [--steps 20] [--group 2] [--resident] --out x.json
then  python tools/tl_bins.py x.json"""
from __future__ import annotations

import argparse
import ctypes
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--group", type=int, default=2)
    ap.add_argument("--streams", type=int, default=8)
    ap.add_argument("--pool", type=int, default=8192)
    ap.add_argument("--resident", action="store_true")
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    import torch
    import paper_2404_00509_b200 as E
    from paper_2404_00509_b200 import _native as N
    path = Path(tempfile.mkdtemp()) / "pool.essl"
    E.build_synthetic(path, args.pool, 256, 95, classes=1000, seed=1)
    cfg = E.LoaderConfig(data=str(path), batch_size=256, res=224, mask_ratio=0.75, out_dtype="bfloat16",
                         resident=args.resident, streams=args.streams, prefetch=args.streams,
                         reuse_outputs=True, group=args.group)
    ld = E.Loader(cfg)
    for k, b in enumerate(ld.epochs(100)):
        if k + 1 >= 3 * args.streams + 3:
            break
    torch.cuda.synchronize()
    ld.set_option(N.ESSL_OPT_PROFILE_KERNELS, 0xFFFF)
    ld.set_option(N.ESSL_OPT_PROFILE, 1)
    ld.profile_read()
    st = torch.cuda.current_stream()
    N.lib().essl_profile_mark(ctypes.c_void_p(st.cuda_stream))
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(st)
    n = 0
    for b in ld.epochs(2, steps=args.steps):
        n += len(b)
    t1.record(st)
    torch.cuda.synchronize()
    total = t0.elapsed_time(t1)
    recs = []
    for s, eng in enumerate(ld.engines):
        for k, a, b in eng.profile_timeline():
            recs.append({"stream": s, "kernel": k, "start": a, "end": b})
    ld.profile_read()
    recs.sort(key=lambda r: r["start"])
    summ = {"steps": args.steps, "group": args.group, "resident": args.resident, "total_ms": total,
            "img_per_s": n / total * 1e3}
    print(json.dumps(summ))
    Path(args.out).write_text(json.dumps({"summary": summ, "launches": recs}))


if __name__ == "__main__":
    main()
