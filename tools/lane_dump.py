"""Per-lane speculative-decode records (ESSL_OPT_DEBUG_LANES) for full-image
crops of a synthetic pool: continuation lengths and merge targets.
    python tools/lane_dump.py [--n 16] [--seq 4096] [--warm 2048]"""
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
    from paper_2404_00509_b200 import _native as N, build
    from paper_2404_00509_b200.engine import Engine
    build.build()
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16)
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--warm", type=int, default=2048)
    ap.add_argument("--pool", default=None)
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    path = Path(args.pool) if args.pool else Path(tempfile.mkdtemp()) / "pool16.essl"
    if not path.exists():
        E.build_synthetic(path, args.n, 256, 95, classes=1000, seed=1)
    h = E.open_container(path)
    n = min(args.n, len(h))
    eng = Engine("cuda:0", max_batch=n, max_side=512, max_payload=h.max_payload())
    eng.set_option(N.ESSL_OPT_SEQ_BITS, args.seq)
    eng.set_option(N.ESSL_OPT_WARMUP_BITS, args.warm)
    eng.set_option(N.ESSL_OPT_DEBUG_LANES, 1)
    blob = h.to_device(eng.device)
    s = eng.samples(n)
    rec = h.records
    s["offset"] = rec["payload_offset"][:n]
    s["length"] = rec["payload_length"][:n]
    s["crc32"] = rec["checksum"][:n]
    s["check_crc"] = 1
    s["w"] = rec["width"][:n]
    s["h"] = rec["height"][:n]
    out = torch.empty((n, 3, 224, 224), dtype=torch.bfloat16, device=eng.device)
    eng.decode_rrc(blob.data_ptr(), s, 224, N.ESSL_OUT_BF16_NCHW, out)
    torch.cuda.synchronize()
    d = np.zeros((n, 64, 8), np.int32)
    N.check(N.lib().essl_debug_lanes(eng._ctx, N.ptr(d), n))
    maxes = []
    for i in range(n):
        nseq = int(d[i, 0, 0])
        L = d[i, :nseq]
        cont = [(int(r[5]) - int(r[1])) for r in L[:nseq - 1] if r[5] >= 0]
        maxes.append(max(cont) if cont else 0)
        print(i, "nseq", nseq, "cont max", max(cont) if cont else 0, "p50", int(np.median(cont)) if cont else 0,
              "top", sorted(cont)[-4:], "nck", [int(x) for x in L[:6, 3]],
              "merge lanes off-by", sorted(set(int(r[7]) - t for t, r in enumerate(L[:nseq - 1]))))
        if args.verbose:
            for t, r in enumerate(L):
                print("   lane", t, r.tolist())
    print(json.dumps({"median_of_max": float(np.median(maxes))}))


if __name__ == "__main__":
    main()
