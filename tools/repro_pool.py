"""Decode a synthetic pool in batches through the Loader and compare each
batch with the C oracle (debug helper).

    python tools/repro_pool.py [--n 1024] [--batch 256] [--side 256] [--q 95] [--seed 3] [--stage 65536]
"""
import argparse
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--side", type=int, default=256)
    ap.add_argument("--q", type=int, default=95)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--stage", type=int, default=65536)
    ap.add_argument("--streams", type=int, default=1)
    args = ap.parse_args()
    import paper_2404_00509_b200 as E
    from paper_2404_00509_b200 import _native as N
    from oracle import oracle as O
    d = Path(tempfile.mkdtemp())
    path = d / "pool.essl"
    E.build_synthetic(path, args.n, args.side, args.q, seed=args.seed)
    cfg = E.LoaderConfig(data=str(path), batch_size=args.batch, res=224, mask_ratio=0.0,
                         streams=args.streams, prefetch=args.streams)
    loader = E.Loader(cfg)
    loader.set_option(N.ESSL_OPT_STAGE_BYTES, args.stage)
    h = loader.handle
    perm = E.epoch_permutation(0, 0, len(h))
    bad = 0
    for s in range(0, len(perm), args.batch):
        idx = perm[s:s + args.batch]
        p = loader.enqueue(0, idx)
        loader.join(p)
        p.event.synchronize()
        res = p.results_host.numpy()
        pix, _, _, st = O.loader_batch(h.bytes, h.records, idx, 0, 0, 224, nthreads=8)
        got = p.batch.pixels.cpu().numpy()
        for i in range(len(idx)):
            if res[i, 0] != st[i] or (st[i] == 0 and not np.array_equal(got[i], pix[i])):
                bad += 1
                if bad <= 10:
                    print("mismatch", int(idx[i]), "gpu status", res[i, :3].tolist(), "oracle", int(st[i]))
    print("batches", -(-len(perm) // args.batch), "mismatches", bad)


if __name__ == "__main__":
    main()
