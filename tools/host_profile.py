"""cProfile of the host side of Loader.epochs (e2e staging path): where the
per-batch Python time goes.  python tools/host_profile.py [--batches 300]"""
from __future__ import annotations

import argparse
import cProfile
import pstats
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
    ap.add_argument("--batches", type=int, default=300)
    ap.add_argument("--resident", action="store_true")
    args = ap.parse_args()
    path = Path(tempfile.mkdtemp()) / "pool.essl"
    E.build_synthetic(path, 8192, 256, 95, classes=1000, seed=1)
    cfg = E.LoaderConfig(data=str(path), batch_size=256, res=224, out_dtype="bfloat16",
                         mask_ratio=0.75, streams=8, prefetch=8, reuse_outputs=True,
                         resident=args.resident)
    loader = E.Loader(cfg)
    for i, b in enumerate(loader.epochs(0)):
        if i >= 40:
            break
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for i, b in enumerate(loader.epochs(1)):
        if i >= args.batches:
            break
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
