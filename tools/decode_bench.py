"""Decode-kernel microbenchmark + per-phase clock breakdown (GPU).

    python tools/decode_bench.py [--n 256] [--side 256] [--q 95] [--sweep]
"""

from __future__ import annotations

import argparse
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

# dbg[0..1]: k_prep start/end; dbg[2..7]: k_entropy PHASE(0..5)
PHASES = ["prep", "hdr_load", "count", "continuation", "resolve", "write_fixup", "p_crc", "p_parse", "p_destuff", "p_tables"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--pool", type=int, default=1024)
    ap.add_argument("--side", type=int, default=256)
    ap.add_argument("--q", type=int, default=95)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("--stage", type=int, default=-1, help="ESSL_OPT_STAGE_BYTES (0: global reader)")
    args = ap.parse_args()
    import torch

    import paper_2404_00509_b200 as E
    from paper_2404_00509_b200 import _native as N
    d = Path(tempfile.mkdtemp())
    path = d / "pool.essl"
    E.build_synthetic(path, args.pool, args.side, args.q, seed=3)
    cfg = E.LoaderConfig(data=str(path), batch_size=args.n, res=224, out_dtype="bfloat16",
                         mask_ratio=0.75, streams=1)
    loader = E.Loader(cfg)
    eng = loader.engine
    if args.stage >= 0:
        eng.set_option(N.ESSL_OPT_STAGE_BYTES, args.stage)
    perm = E.epoch_permutation(0, 0, len(loader.handle))
    settings = [("spec", 4096, 2048)]
    if args.sweep:
        settings = [("serial", 0, 0)] + [("spec", s, w) for s in (2048, 4096, 8192)
                                         for w in (0, 1024, 2048, 4096)]
    results = []
    for mode, sb, ov in settings:
        eng.set_option(N.ESSL_OPT_DECODE_MODE, N.ESSL_DECODE_SERIAL if mode == "serial"
                       else N.ESSL_DECODE_SPECULATIVE)
        if mode == "spec":
            eng.set_option(N.ESSL_OPT_SEQ_BITS, sb)
            eng.set_option(N.ESSL_OPT_WARMUP_BITS, ov)
        idx = perm[:args.n]
        loader.finish(loader.enqueue(0, idx))  # warm
        eng.set_option(N.ESSL_OPT_PROFILE, 1)
        eng.profile_read()
        for r in range(args.reps):
            loader.finish(loader.enqueue(0, perm[(r * args.n) % len(perm):][:args.n]))
        prof = eng.profile_read()
        eng.set_option(N.ESSL_OPT_PROFILE, 0)
        dbg = np.zeros(16 * args.n, np.int64)
        N.check(N.lib().essl_debug_stats(eng._ctx, N.ptr(dbg), args.n))
        dbg = dbg.reshape(args.n, 16)
        ph = np.stack([dbg[:, 1] - dbg[:, 0]] + [dbg[:, 3 + i] - dbg[:, 2 + i] for i in range(5)]
                      + [dbg[:, 13] - dbg[:, 12], dbg[:, 14] - dbg[:, 13], dbg[:, 15] - dbg[:, 14],
                         dbg[:, 1] - dbg[:, 15]], 1)
        nseq = dbg[:, 10] & 0xFFFFFFFF
        ext = dbg[:, 10] >> 32
        cont = dbg[:, 11]
        row = {"mode": mode, "seq_bits": sb, "warm_bits": ov,
               "decode_ms": prof["decode"][0] / prof["decode"][1],
               "resize_ms": prof.get("resize", (0, 1))[0] / max(prof.get("resize", (0, 1))[1], 1),
               "phase_kcycles_median": {PHASES[i]: round(float(np.median(ph[:, i])) / 1e3, 1)
                                        for i in range(10)},
               "phase_kcycles_max": {PHASES[i]: round(float(np.max(ph[:, i])) / 1e3, 1)
                                     for i in range(10)},
               "units_phase1_mean": float((dbg[:, 8] & 0xFFFFFFFF).mean()),
               "reguess_phase1_mean": float((dbg[:, 8] >> 32).mean()),
               "units_phase1_lane_max_median": float(np.median(dbg[:, 9] & 0xFFFFFFFF)),
               "fallback_images": int((dbg[:, 9] >> 32).sum()),
               "nseq_mean": float(nseq.mean()), "extended_images": int((ext > 0).sum()),
               "cont_bits_max_median": float(np.median(cont)),
               "cont_bits_max_max": int(cont.max())}
        results.append(row)
        print(json.dumps(row), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(results, indent=1))
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
