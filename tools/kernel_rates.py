"""Per-kernel throughput at full occupancy: one stream, one big batch (so
every launch fills the GPU), each kernel bracketed by CUDA events
(ESSL_OPT_PROFILE, all kernels).  Analysis tool, not a benchmark:
    python tools/kernel_rates.py [--n 2048] [--reps 5]"""
from __future__ import annotations

import argparse
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--pool", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--tag", default="")
    ap.add_argument("--warm", type=int, default=-1, help="ESSL_OPT_WARMUP_BITS (-1: default)")
    ap.add_argument("--seq", type=int, default=0, help="ESSL_OPT_SEQ_BITS (0: default)")
    args = ap.parse_args()
    import paper_2404_00509_b200 as E
    from paper_2404_00509_b200 import _native as N
    path = Path(tempfile.mkdtemp()) / "pool.essl"
    E.build_synthetic(path, args.pool, 256, 95, classes=1000, seed=1)
    cfg = E.LoaderConfig(data=str(path), batch_size=args.n, res=224, out_dtype="bfloat16",
                         mask_ratio=0.75, streams=1, prefetch=1)
    loader = E.Loader(cfg)
    eng = loader.engine
    if args.warm >= 0:
        eng.set_option(N.ESSL_OPT_WARMUP_BITS, args.warm)
    if args.seq > 0:
        eng.set_option(N.ESSL_OPT_SEQ_BITS, args.seq)
    perm = E.epoch_permutation(0, 0, len(loader.handle))

    def run(r):  # (analysis builds may produce bad statuses: timing only)
        p = loader.enqueue(0, perm[(r * args.n) % len(perm):][:args.n])
        try:
            loader.finish(p)
        except Exception as exc:  # noqa: BLE001
            out.setdefault("errors", str(exc)[:80])
    out = {"tag": args.tag, "n": args.n, "warm": args.warm, "seq": args.seq}
    for r in range(2):
        run(r)
    eng.set_option(N.ESSL_OPT_PROFILE_KERNELS, 0xFFFF)
    eng.set_option(N.ESSL_OPT_PROFILE, 1)
    eng.profile_read()
    for r in range(args.reps):
        run(r)
    prof = eng.profile_read()
    eng.set_option(N.ESSL_OPT_PROFILE, 0)
    for k, (ms, c) in prof.items():
        if k == "decode":
            continue
        per = ms / c
        out[k] = {"ms": round(per, 4), "img_per_s": round(args.n / per * 1e3)}
    import numpy as np
    dbg = np.zeros(16 * args.n, np.int64)
    N.check(N.lib().essl_debug_stats(eng._ctx, N.ptr(dbg), args.n))
    dbg = dbg.reshape(args.n, 16)
    # k_entropy PHASE(0..5) clocks in dbg[2..7]: prologue, phase 1, continuation,
    # resolution, block tables
    names = ["prologue", "phase1", "continuation", "resolution", "tables"]
    ph = np.stack([dbg[:, 3 + i] - dbg[:, 2 + i] for i in range(5)], 1)
    out["entropy_phase_kcycles"] = {names[i]: [round(float(np.percentile(ph[:, i], q)) / 1e3, 1)
                                               for q in (10, 50, 90, 100)] for i in range(5)}
    pn = ["load", "crc", "parse", "destuff", "tables"]
    pp = np.stack([dbg[:, 12] - dbg[:, 0], dbg[:, 13] - dbg[:, 12], dbg[:, 14] - dbg[:, 13],
                   dbg[:, 15] - dbg[:, 14], dbg[:, 1] - dbg[:, 15]], 1)
    out["prep_phase_kcycles"] = {pn[i]: [round(float(np.percentile(pp[:, i], q)) / 1e3, 1)
                                         for q in (10, 50, 90)] for i in range(5)}
    out["extended_images_frac"] = round(float(((dbg[:, 10] >> 32) > 0).mean()), 4)
    out["fallback_images"] = int((dbg[:, 9] >> 32).sum())
    out["entropy_cta_kcycles"] = [round(float(np.percentile(dbg[:, 7] - dbg[:, 2], q)) / 1e3, 1)
                                  for q in (10, 50, 90, 100)]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
