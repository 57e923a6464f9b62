"""The pipelined loader with the host taken out: `--batches` consecutive
batches of the bench workload (6 streams, HBM-resident) captured once into a
CUDA graph through Loader.enqueue, then replayed.  Reports the replay's
images/s (device time, no host enqueue cost) and, with
ESSL_PROFILER_RANGE=1, brackets one replay with cudaProfilerStart/Stop so
`ncu --replay-mode app-range` measures the concurrent kernel mix as one range
(SM pipe utilisation, issue activity, warp states of the real pipeline).
Analysis tool, not the product path (the graph replays the captured
descriptors).

    python tools/graph_profile.py [--streams 6] [--batches 48]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch
    import paper_2404_00509_b200 as E
    from paper_2404_00509_b200 import build
    build.build()
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=6)
    ap.add_argument("--batches", type=int, default=48)
    ap.add_argument("--pool", type=int, default=4096)
    ap.add_argument("--replays", type=int, default=5)
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
    for i in range(4 * args.streams):  # warm-up: contexts, output ring, attributes
        pend.append(loader.enqueue(0, perm[(i % nb) * 256:][:256]))
    for p in pend:
        loader.finish(p)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        pend = [loader.enqueue(0, perm[(i % nb) * 256:][:256]) for i in range(args.batches)]
        for p in pend:
            loader.join(p)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    torch.cuda.synchronize()
    ms = []
    for _ in range(args.replays):
        a.record(st)
        g.replay()
        b.record(st)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    if os.environ.get("ESSL_PROFILER_RANGE") == "1":
        torch.cuda.cudart().cudaProfilerStart()
        g.replay()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
    best = min(ms)
    print(json.dumps({"streams": args.streams, "batches": args.batches,
                      "ms_per_replay": [round(x, 3) for x in ms],
                      "img_per_s": round(args.batches * 256 / best * 1e3)}))


if __name__ == "__main__":
    main()
