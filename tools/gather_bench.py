"""Host->device payload gather (essl_stage_pinned) bandwidth in isolation:
one batch of the bench pool's payloads per launch, CUDA-event timed, over
ESSL_OPT_GATHER_CTAS x ESSL_OPT_GATHER_TMA.  Analysis tool:
    python tools/gather_bench.py [--batch 256] [--ctas 4 8 16 32]"""
from __future__ import annotations

import argparse
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--pool", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ctas", type=int, nargs="+", default=[1, 2, 4, 8, 16, 32, 64])
    args = ap.parse_args()
    import torch
    import paper_2404_00509_b200 as E
    from paper_2404_00509_b200 import _native as N
    path = Path(tempfile.mkdtemp()) / "pool.essl"
    E.build_synthetic(path, args.pool, 256, 95, classes=1000, seed=1)
    cfg = E.LoaderConfig(data=str(path), batch_size=args.batch, res=224, resident=False, streams=1)
    ld = E.Loader(cfg)
    eng = ld.engine
    rec = ld.handle.records
    perm = E.epoch_permutation(0, 0, len(ld.handle))
    st = torch.cuda.current_stream()
    out = []
    for tma in (1, 0):
        for ctas in args.ctas:
            eng.set_option(N.ESSL_OPT_GATHER_CTAS, ctas)
            eng.set_option(N.ESSL_OPT_GATHER_TMA, tma)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            nbytes = 0
            for r in range(args.reps + 2):
                idx = perm[(r * args.batch) % len(perm):][:args.batch]
                samples = np.zeros(len(idx), N._np_dtypes()[0])
                off = rec["payload_offset"][idx].astype(np.uint64)
                ln = rec["payload_length"][idx].astype(np.uint32)
                if r == 2:
                    torch.cuda.synchronize()
                    a.record(st)
                if r >= 2:
                    nbytes += int(ln.sum())
                eng.stage_pinned(r & 1, ld._pinned_base, off, ln, samples, st)
            b.record(st)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            row = {"tma": tma, "ctas": ctas, "ms_per_batch": round(ms / args.reps, 4),
                   "GBps": round(nbytes / ms / 1e6, 2)}
            print(json.dumps(row), flush=True)
            out.append(row)


if __name__ == "__main__":
    main()
