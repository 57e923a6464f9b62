"""Host->device payload paths, timed alone (CUDA events):
  gather : essl_stage_pinned (k_host_gather reading the page-locked container)
  stage  : essl_stage (host threads gather into the pinned ring + one H2D copy)
  copy   : one contiguous cudaMemcpyAsync of the same byte count (copy-engine bound)
Usage: python tools/h2d_bench.py [--batch 256] [--iters 50]"""

from __future__ import annotations

import argparse
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch
    import paper_2404_00509_b200 as E
    from paper_2404_00509_b200 import build
    from paper_2404_00509_b200.engine import Engine
    build.build()
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--pool", type=int, default=8192)
    ap.add_argument("--gather-ctas", type=int, nargs="*", default=[0, 8, 16, 32])
    args = ap.parse_args()
    d = Path(tempfile.mkdtemp())
    path = d / "pool.essl"
    E.build_synthetic(path, args.pool, 256, 95, classes=1000, seed=1)
    h = E.open_container(path)
    rec = h.records
    base = h.pinned_host()
    eng = Engine("cuda:0", max_batch=args.batch, max_side=256, max_payload=h.max_payload())
    st = torch.cuda.Stream()
    rng = np.random.default_rng(0)
    out = {}

    def timed(fn, nbytes):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(args.iters):
            fn()
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.iters
        return {"ms": ms, "GBps": nbytes / ms / 1e6}

    idx = rng.permutation(len(h))[:args.batch]
    offs = np.ascontiguousarray(rec["payload_offset"][idx], np.uint64)
    lens = np.ascontiguousarray(rec["payload_length"][idx], np.uint32)
    nbytes = int(lens.sum())
    s = eng.samples(args.batch)
    slot = [0]

    def gather():
        eng.stage_pinned(slot[0], base, offs, lens.copy(), s, stream=st)
        slot[0] ^= 1
    from paper_2404_00509_b200 import _native as N
    for tma in (0, 1):
        eng.set_option(N.ESSL_OPT_GATHER_TMA, tma)
        for g in args.gather_ctas:
            eng.set_option(N.ESSL_OPT_GATHER_CTAS, g)
            out[f"gather{'_tma' if tma else ''}_{g}"] = timed(gather, nbytes)
    eng.set_option(N.ESSL_OPT_GATHER_TMA, 0)

    ptrs = (np.frombuffer(h.bytes, np.uint8).ctypes.data + offs).astype(np.uint64)

    def stage():
        eng.stage(slot[0], ptrs, lens, s, nthreads=8, stream=st)
        slot[0] ^= 1
    out["stage"] = timed(stage, nbytes)

    src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")

    def copy():
        with torch.cuda.stream(st):
            dst.copy_(src, non_blocking=True)
    out["copy"] = timed(copy, nbytes)
    out["bytes_per_batch"] = nbytes
    print(json.dumps(out))


if __name__ == "__main__":
    main()
