"""Host cost of one batch enqueue (Loader.enqueue -> essl_batch_enqueue) on
the bench workload: the whole Python call, the native call alone, and the
native RRC draws alone.  python tools/enqueue_profile.py [--n 200]"""
import argparse
import ctypes
import json
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch
    import paper_2404_00509_b200 as E
    from paper_2404_00509_b200 import _native as N
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200)
    args = ap.parse_args()
    path = Path(tempfile.mkdtemp()) / "p.essl"
    E.build_synthetic(path, 2048, 256, 95, classes=1000, seed=1)
    cfg = E.LoaderConfig(data=str(path), batch_size=256, res=224, mask_ratio=0.75,
                         out_dtype="bfloat16", streams=8, prefetch=8, reuse_outputs=True)
    ld = E.Loader(cfg)
    perm = E.epoch_permutation(0, 0, 2048)
    idx = [np.ascontiguousarray(perm[(i * 256) % 2048:][:256]) for i in range(8)]
    pend = [ld.enqueue(0, idx[i % 8]) for i in range(32)]
    for p in pend:
        ld.finish(p)
    torch.cuda.synchronize()
    # the native call alone, timed inside the Python enqueue
    lib = N.lib()
    native_fn = lib.essl_batch_enqueue
    tn = []

    class _Timed:
        def __call__(self, *a):
            t0 = time.perf_counter()
            r = native_fn(*a)
            tn.append(time.perf_counter() - t0)
            return r
    lib.essl_batch_enqueue = _Timed()
    # whole Python enqueue
    t = []
    pend = []
    for i in range(args.n):
        t0 = time.perf_counter()
        pend.append(ld.enqueue(0, idx[i % 8]))
        t.append(time.perf_counter() - t0)
        if len(pend) > 16:
            ld.finish(pend.pop(0))
    for p in pend:
        ld.finish(p)
    torch.cuda.synchronize()
    # native RRC draws alone
    s = np.zeros(256, N._np_dtypes()[0])
    w = ld._widths
    h = ld._heights
    r = []
    for i in range(args.n):
        t0 = time.perf_counter()
        N.lib().essl_rrc_batch(0, i, N.ptr(idx[i % 8]), 256, N.ptr(w), N.ptr(h), 0.08, 1.0, 0.75,
                               4 / 3, N.ptr(s))
        r.append(time.perf_counter() - t0)
    lib.essl_batch_enqueue = native_fn
    out = {"enqueue_ms_median": 1e3 * float(np.median(t)), "enqueue_ms_p90": 1e3 * float(np.percentile(t, 90)),
           "native_call_ms_median": 1e3 * float(np.median(tn)),
           "rrc_batch_ms_median": 1e3 * float(np.median(r))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
