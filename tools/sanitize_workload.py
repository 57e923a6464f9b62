"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): the
smoke batch plus one bench-shaped batch (64 x 256px q95, mask 0.75, visible
tokens), a host-staged batch, a restart-marker batch and a 3-Aug+ batch, all
checked against the oracle so a sanitizer run is also a parity run.

    compute-sanitizer --tool memcheck python tools/sanitize_workload.py
"""
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch
    import __graft_entry__ as G
    G.smoke()
    import paper_2404_00509_b200 as E
    from oracle import oracle as O
    d = Path(tempfile.mkdtemp())
    E.build_synthetic(d / "a.essl", 64, 256, 95, seed=3)
    E.build_synthetic(d / "r.essl", 16, 256, 90, seed=4, restart_interval=4)
    for path, kw in ((d / "a.essl", dict(mask_ratio=0.75, visible=True, out_dtype="bfloat16")),
                     (d / "a.essl", dict(resident=False, mask_ratio=0.75)),
                     (d / "r.essl", dict()),
                     (d / "a.essl", dict(aug="3aug+"))):
        with E.open_container(path) as h:
            cfg = E.LoaderConfig(data=str(path), batch_size=64, res=224, streams=2, prefetch=2,
                                 **kw)
            loader = E.Loader(cfg, container=h)
            b = next(iter(loader.epoch(0)))
            torch.cuda.synchronize()
            idx = b.indices.cpu().numpy()
            pix, _, _, st = O.loader_batch(h.bytes, h.records, idx, 0, 0, 224,
                                           mask_ratio=kw.get("mask_ratio", 0.0),
                                           aug=kw.get("aug", "simple"))
            assert (st == 0).all()
            got = b.pixels.float().cpu().numpy()
            assert np.abs(got - pix).max() <= 1e-2, kw
            loader.close()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
