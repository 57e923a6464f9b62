"""Throughput of the UNMODIFIED reference loader (cropload.pipeline.Loader,
installed under baseline/_ref with `pip install --target`) on this host's
cores, over the same container the GPU bench reads.

    python tools/ref_loader_rate.py --data pool.essl --batch 256 --mask 0.75 \
        --seconds 8 --mode threads|single|procs

threads: Loader(workers=os.cpu_count()) through Loader.epoch (the primary
         CPU baseline; thread scaling is GIL-bound);
single : Loader(workers=1) (the per-core rate);
procs  : one process per core, each filling its own disjoint share of the
         epoch's samples with the reference's per-sample code
         (Loader._fill_sample, the body of Loader.epoch), throughput summed
         (the process-parallel upper bound).
One JSON line on stdout.  Numba compiles the reference kernels on first use
(NUMBA_CACHE_DIR caches them); that warm-up is outside the timed region.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"


def _import_ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/essl_numba_cache")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import cropload.pipeline as P  # noqa: F401  (the reference package)
    return P


def _cfg(P, args, workers):
    return P.LoaderConfig(data=args.data, batch_size=args.batch, workers=workers, seed=0,
                          res=args.res, scale=tuple(args.scale), mask_ratio=args.mask)


def run_epoch_mode(args, workers) -> dict:
    P = _import_ref()
    with P.Loader(_cfg(P, args, workers)) as loader:
        it = loader.epoch(0)
        next(it)  # numba JIT + thread pool warm-up
        n, t0 = 0, time.perf_counter()
        e = 1
        while True:
            for b in it:
                n += len(b.labels)
                if time.perf_counter() - t0 >= args.seconds:
                    break
            el = time.perf_counter() - t0
            if el >= args.seconds:
                break
            it = loader.epoch(e)
            e += 1
    return {"value": n / el, "images": n, "seconds": el, "workers": workers}


def _proc_worker(args, rank, nproc, q, start_evt):
    P = _import_ref()
    import numpy as np
    loader = P.Loader(_cfg(P, args, 1))
    perm = P.epoch_permutation(0, 0, len(loader.handle))
    mine = perm[rank::nproc]
    res = args.res
    k = loader.mask_spec.masked_count if loader.mask_spec is not None else 0

    def new_batch(b):
        return P.ImageBatch(pixels=np.empty((b, 3, res, res), np.float32),
                            labels=np.empty(b, np.int64), indices=np.empty(b, np.int64), epoch=0,
                            mask=np.empty((b, k), np.int32) if k else None, uint8=None)

    batch = new_batch(args.batch)
    for slot, idx in enumerate(mine[:8]):  # JIT warm-up
        loader._fill_sample(0, int(idx), batch, slot % args.batch)
    q.put(("ready", rank))
    start_evt.wait()
    n, t0, i = 0, time.perf_counter(), 0
    while time.perf_counter() - t0 < args.seconds:
        idx = int(mine[i % len(mine)])
        loader._fill_sample(0, idx, batch, i % args.batch)
        n += 1
        i += 1
    q.put(("done", n, time.perf_counter() - t0))


def run_procs(args) -> dict:
    nproc = os.cpu_count() or 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    start = ctx.Event()
    ps = [ctx.Process(target=_proc_worker, args=(args, r, nproc, q, start)) for r in range(nproc)]
    for p in ps:
        p.start()
    for _ in ps:
        q.get(timeout=600)
    start.set()
    tot, secs = 0, []
    for _ in ps:
        _, n, s = q.get(timeout=600)
        tot += n
        secs.append(s)
    for p in ps:
        p.join(timeout=60)
    return {"value": tot / max(secs), "images": tot, "seconds": max(secs), "processes": nproc}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--data", required=True)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--res", type=int, default=224)
    ap.add_argument("--scale", type=float, nargs=2, default=(0.08, 1.0))
    ap.add_argument("--mask", type=float, default=0.75)
    ap.add_argument("--seconds", type=float, default=8.0)
    ap.add_argument("--mode", default="threads", choices=["threads", "single", "procs"])
    args = ap.parse_args()
    if not (REF / "cropload").exists():
        print(json.dumps({"mode": args.mode, "unavailable": f"{REF} not installed"}))
        return
    if args.mode == "procs":
        r = run_procs(args)
    else:
        r = run_epoch_mode(args, os.cpu_count() or 1 if args.mode == "threads" else 1)
    r.update(mode=args.mode, unit="images/s", cpu=_cpu_model(), cores=os.cpu_count())
    print(json.dumps(r), flush=True)


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


if __name__ == "__main__":
    main()
