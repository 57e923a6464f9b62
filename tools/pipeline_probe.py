"""Which stage bounds the pipelined throughput?  Runs the bench-shaped loader
loop (6 streams, batches of 256 cfg2 images, HBM-resident) with stages
removed (analysis only; not a benchmark of the product path):
    python tools/pipeline_probe.py --variant full|no_mask|no_resize|decode_only"""
from __future__ import annotations

import argparse
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch
    import paper_2404_00509_b200 as E
    from paper_2404_00509_b200 import _native as N, build
    build.build()
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="full")
    ap.add_argument("--streams", type=int, default=6)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--pool", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--depth", type=int, default=2, help="pending batches per stream")
    args = ap.parse_args()
    path = Path(tempfile.mkdtemp()) / "pool.essl"
    E.build_synthetic(path, args.pool, 256, 95, classes=1000, seed=1)
    mask = 0.0 if args.variant in ("no_mask", "decode_only") else 0.75
    cfg = E.LoaderConfig(data=str(path), batch_size=args.batch, res=224, out_dtype="bfloat16",
                         mask_ratio=mask, streams=args.streams, prefetch=args.streams,
                         reuse_outputs=True)
    loader = E.Loader(cfg)
    if args.variant in ("no_resize", "decode_only"):
        for eng in loader.engines:
            orig = eng.decode_rrc

            def dr(blob, samples, res, kind, out=None, u8=None, results=None, stream=None,
                   max_side=0, aug=None, _o=orig):
                return _o(blob, samples, res, N.ESSL_OUT_NONE, None, None, results, stream,
                          max_side, aug)
            eng.decode_rrc = dr
    perm = E.epoch_permutation(0, 0, len(loader.handle))
    B = args.batch
    nb = len(perm) // B
    pend = []
    for i in range(30):
        pend.append(loader.enqueue(0, perm[(i % nb) * B:][:B]))
        if len(pend) > args.depth * args.streams:
            loader.finish(pend.pop(0))
    for p in pend:
        loader.finish(p)
    import gc
    gc.collect()
    gc.freeze()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    pend = []
    import time
    hs = []
    for i in range(args.steps):
        h0 = time.perf_counter()
        pend.append(loader.enqueue(0, perm[(i % nb) * B:][:B]))
        hs.append(time.perf_counter() - h0)
        if len(pend) > args.depth * args.streams:
            loader.finish(pend.pop(0))
    for p in pend:
        loader.join(p)
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    import numpy as np
    print(json.dumps({"variant": args.variant, "streams": args.streams, "batch": B,
                      "ms_per_batch": round(ms, 4), "img_per_s": round(B / ms * 1e3),
                      "host_enqueue_ms_median": round(float(np.median(hs)) * 1e3, 4)}))


if __name__ == "__main__":
    main()
