"""Generate the committed golden fixtures from the REFERENCE implementation.

Run in the build container (the reference is importable there, it is not on
the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Every input (containers, JPEG streams, RGB arrays) is produced by the
reference's own fixture generators (``cropload.synth.write_corpus``,
``cropload.container.build_container``, ``cropload.jpeg.encode_jpeg``) or by
Pillow (external-codec streams, as in the reference's test_jpeg.py:246-274).
Every expected output is computed by the reference's own functions.  Large
outputs are stored as SHA-256 digests of their raw bytes; small ones (rects,
masks, permutations, coefficient windows of a few streams) verbatim.

Outputs (all under tests/golden/):
    *.essl            reference-format containers (container.py:1-20)
    streams/*.jpg     individual JPEG streams
    golden.json       expected values / digests
    arrays.npz        verbatim arrays
"""

from __future__ import annotations

import hashlib
import io
import json
import shutil
import sys
import zlib
import tempfile
from pathlib import Path

import numpy as np

from cropload import imgops, masking, rng as R
from cropload.container import BuildSpec, build_container, open_container
from cropload.errors import CroploadError
from cropload.jpeg import CropRect, decode_crop, decode_full, encode_jpeg
from cropload.jpeg import codec as C
from cropload.jpeg import tables as T
from cropload.jpeg.decode_kernels import decode_scan_baseline
from cropload.pipeline import Loader, LoaderConfig, RrcConfig, sample_rrc
from cropload.schedule import builtin_scheme, load_scheme, params_for_epoch
from cropload.synth import synth_image, write_corpus

OUT = Path(__file__).resolve().parent


def sha(a) -> str:
    if isinstance(a, (bytes, bytearray)):
        return hashlib.sha256(a).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_coefs(data: bytes, rect: CropRect):
    """The int32 coefficient arrays decode_crop holds before reconstruction
    (codec.py:471-500): rows < row_stop decoded, the rest zero."""
    arr = np.frombuffer(data, np.uint8)
    frame = C.parse_stream(data)
    rect.validate(frame.width, frame.height)
    scan = frame.scans[0]
    gx, gy, units = C._scan_units(frame, scan)
    if len(frame.comps) > 1:
        mcu_h = 8 * frame.vmax
    else:
        mcu_h = 8
    my1 = (rect.y + rect.h - 1) // mcu_h
    coefs = C._alloc_coefs(frame)
    max_restarts = (gx * gy) // scan.ri if scan.ri else 0
    clean, restarts, nr = C._destuff(arr, scan, max_restarts)
    ns = len(scan.slots)
    luts = C._lut_stack([s[1] for s in scan.slots] + [s[2] for s in scan.slots])
    c0 = coefs[0]
    c1 = coefs[1] if len(coefs) > 1 else coefs[0][:1, :1]
    c2 = coefs[2] if len(coefs) > 2 else coefs[0][:1, :1]
    st, vpos, cnt = decode_scan_baseline(
        clean, restarts, nr, scan.ri, luts, np.arange(ns, dtype=np.int64),
        np.arange(ns, 2 * ns, dtype=np.int64),
        np.array([u[0] for u in units], np.int64), np.array([u[1] for u in units], np.int64),
        np.array([u[2] for u in units], np.int64), ns, gx, my1 + 1, c0, c1, c2,
        T.ZIGZAG_TO_NATURAL)
    assert st == 0
    return coefs


def build_fixture_container(name, n, classes, min_side, max_side, seed, max_res, q):
    tmp = Path(tempfile.mkdtemp())
    write_corpus(tmp / "src", n, classes=classes, min_side=min_side,
                 max_side=max_side, seed=seed)
    out = OUT / name
    build_container(BuildSpec(tmp / "src", max_res, q, seed=seed), out, workers=4)
    shutil.rmtree(tmp)
    return out


def loader_golden(path: Path, cfg_kw: dict, epochs=(0,)):
    """Run the reference Loader and record per-sample digests."""
    recs = []
    cfg = LoaderConfig(data=str(path), workers=2, **cfg_kw)
    with Loader(cfg) as loader:
        h = loader.handle
        for e in epochs:
            for b in loader.epoch(e):
                for s in range(len(b)):
                    idx = int(b.indices[s])
                    rng = R.SampleRng(cfg.seed, e, idx, R.DOMAIN_PIPELINE)
                    _, w, hh, _ = h.read_sample(idx)
                    r = sample_rrc(rng, w, hh, loader.rrc)
                    flip = int(rng.random() < 0.5)
                    recs.append({
                        "epoch": e, "index": idx, "label": int(b.labels[s]),
                        "rect": [r.x, r.y, r.w, r.h], "flip": flip,
                        "pixels": sha(b.pixels[s]),
                        "uint8": sha(b.uint8[s]) if b.uint8 is not None else None,
                        "mask": b.mask[s].tolist() if b.mask is not None else None,
                    })
    return recs


def main():
    g: dict = {"generator": "tests/golden/make_golden.py (reference cropload 0.1.0)"}
    arrays: dict = {}

    # ---- containers -------------------------------------------------------
    cfg1 = build_fixture_container("cfg1_small.essl", 16, 4, 256, 256, 1, 256, 95)
    cfg4 = build_fixture_container("cfg4_small.essl", 4, 2, 512, 512, 1, 512, 90)
    mixed = build_fixture_container("mixed_small.essl", 12, 3, 120, 420, 11, 384, 90)

    g["containers"] = {}
    for p in (cfg1, cfg4, mixed):
        with open_container(p) as h:
            recs = h.records
            g["containers"][p.name] = {
                "count": len(h), "file_sha": sha(p.read_bytes()),
                "payload_length": recs["payload_length"].tolist(),
                "width": recs["width"].tolist(), "height": recs["height"].tolist(),
                "label": recs["label"].tolist(), "checksum": recs["checksum"].tolist(),
            }

    # ---- loader end-to-end ------------------------------------------------
    g["loader"] = {
        "cfg1_simple_224": {"data": cfg1.name, "cfg": dict(batch_size=8, seed=0, res=224),
                            "epochs": [0, 1]},
        "cfg1_mask_224": {"data": cfg1.name, "cfg": dict(batch_size=8, seed=0, res=224,
                                                         mask_ratio=0.75, patch=16,
                                                         keep_uint8=True), "epochs": [0]},
        "cfg4_pt_224": {"data": cfg4.name, "cfg": dict(batch_size=4, seed=3, res=224,
                                                       scale=(0.2, 1.0)), "epochs": [0, 2]},
        "mixed_96_u8": {"data": mixed.name, "cfg": dict(batch_size=5, seed=77, res=96,
                                                        keep_uint8=True), "epochs": [4]},
    }
    # cfg3: progressive resolution 112 -> 160 -> 192 -> 224 (schedule.py:198-223)
    scheme_doc = {"name": "prog4", "stages": [
        {"res": r, "m": 0.75, "aug": "simple", "sigma": [0.2 ** 0.5, 1.0], "span": 0.25}
        for r in (112, 160, 192, 224)]}
    scheme = load_scheme(scheme_doc)
    g["scheme_prog4"] = scheme_doc
    for e in (0, 1, 2, 3):
        p = params_for_epoch(scheme, e, 4)
        g["loader"][f"cfg3_epoch{e}"] = {
            "data": cfg1.name, "epochs": [e],
            "cfg": dict(batch_size=8, seed=0, res=p.resolution,
                        scale=p.scale.area_bounds(), mask_ratio=p.masking_ratio,
                        patch=16)}
    for key, spec in g["loader"].items():
        spec["samples"] = loader_golden(OUT / spec["data"], spec["cfg"], spec["epochs"])
        spec["cfg"] = {k: (list(v) if isinstance(v, tuple) else v) for k, v in spec["cfg"].items()}
        print(key, len(spec["samples"]), file=sys.stderr)

    # ---- codec streams ----------------------------------------------------
    sdir = OUT / "streams"
    sdir.mkdir(exist_ok=True)
    streams = {}
    rngc = np.random.default_rng(5)
    corpus = []
    for i in range(6):
        hh = int(rngc.integers(120, 420)); ww = int(rngc.integers(120, 420))
        corpus.append(synth_image(7000 + i, hh, ww))
    streams["q85_rst7"] = encode_jpeg(corpus[0], 85, restart_interval=7)
    streams["q85_rst1"] = encode_jpeg(corpus[1], 85, restart_interval=1)
    streams["q92"] = encode_jpeg(corpus[2], 92)
    streams["q100"] = encode_jpeg(synth_image(55, 256, 256), 100)
    streams["q50_odd"] = encode_jpeg(synth_image(3, 37, 61), 50)
    streams["white_1x1"] = encode_jpeg(np.full((1, 1, 3), 255, np.uint8), 90)
    streams["flat_64"] = encode_jpeg(np.full((64, 64, 3), 128, np.uint8), 95)
    img6 = synth_image(6, 150, 200)
    from PIL import Image
    for nm, kw in (("pil_444", {"subsampling": 0}), ("pil_422", {"subsampling": 1}),
                   ("pil_420_opt", {"subsampling": 2, "optimize": True})):
        buf = io.BytesIO()
        Image.fromarray(img6).save(buf, "JPEG", quality=88, **kw)
        streams[nm] = buf.getvalue()
    buf = io.BytesIO()
    Image.fromarray(img6).convert("L").save(buf, "JPEG", quality=88)
    streams["pil_gray"] = buf.getvalue()
    buf = io.BytesIO()
    Image.fromarray(synth_image(4, 180, 140)).save(buf, "JPEG", quality=90, progressive=True)
    streams["pil_progressive"] = buf.getvalue()
    streams["truncated_half"] = streams["q92"][:len(streams["q92"]) // 2]
    streams["truncated_hdr"] = streams["q92"][:40]
    streams["not_jpeg"] = b"not a jpeg at all"

    g["streams"] = {}
    for nm, data in streams.items():
        (sdir / f"{nm}.jpg").write_bytes(data)
        ent = {"sha": sha(data), "crops": []}
        try:
            full, st = decode_full(data)
            ent["full"] = {"sha": sha(full), "shape": list(full.shape),
                           "stats": [st.mcus_entropy_decoded, st.mcus_reconstructed,
                                     bool(st.fallback_full)]}
            hgt, wid = full.shape[:2]
            rr = np.random.default_rng(zlib.crc32(nm.encode()))
            rects = [(0, 0, wid, hgt)]
            for _ in range(12):
                cw = int(rr.integers(1, wid + 1)); ch = int(rr.integers(1, hgt + 1))
                rects.append((int(rr.integers(0, wid - cw + 1)),
                              int(rr.integers(0, hgt - ch + 1)), cw, ch))
            for (x, y, cw, ch) in rects:
                crop, cs = decode_crop(data, CropRect(x, y, cw, ch))
                c = {"rect": [x, y, cw, ch], "sha": sha(crop),
                     "stats": [cs.mcus_entropy_decoded, cs.mcus_reconstructed,
                               bool(cs.fallback_full)]}
                if not cs.fallback_full:
                    co = ref_coefs(data, CropRect(x, y, cw, ch))
                    c["coef_sha"] = [sha(a) for a in co]
                ent["crops"].append(c)
            # out-of-bounds rects (test_jpeg.py:173-179)
            ent["bad_rects"] = [[0, 0, wid + 1, hgt], [-1, 0, 4, 4],
                                [wid - 2, 0, 3, 1], [0, hgt, 1, 1]]
            for br in ent["bad_rects"]:
                try:
                    decode_crop(data, CropRect(*br))
                    raise AssertionError("expected ValueError")
                except ValueError:
                    pass
        except CroploadError as exc:
            ent["error"] = {"type": type(exc).__name__, "msg": str(exc),
                            "offset": getattr(exc, "offset", None)}
        g["streams"][nm] = ent
    # a verbatim coefficient window for one stream (debug aid)
    co = ref_coefs(streams["q92"], CropRect(10, 20, 60, 40))
    arrays["coefs_q92_y"] = co[0][:6]

    # ---- pixel ops ----------------------------------------------------------
    rr = np.random.default_rng(17)
    g["resize"] = []
    for i, (ih, iw, oh, ow) in enumerate(((37, 61, 224, 224), (100, 40, 64, 64),
                                         (224, 224, 160, 160), (9, 9, 32, 32),
                                         (256, 200, 112, 112), (23, 31, 48, 16))):
        src = rr.integers(0, 256, (ih, iw, 3), dtype=np.uint8)
        arrays[f"resize_src_{i}"] = src
        g["resize"].append({"in": [ih, iw], "out": [oh, ow],
                            "sha": sha(imgops.resize_bilinear(src, oh, ow))})
    src = np.zeros((2, 2, 3), np.uint8)
    src[:, 1] = 255
    g["resize_2x2_row"] = imgops.resize_bilinear(src, 4)[0, :, 0].astype(int).tolist()
    nimg = rr.integers(0, 256, (50, 70, 3), dtype=np.uint8)
    arrays["normalize_src"] = nimg
    g["normalize_sha"] = sha(imgops.normalize(nimg))
    g["normalize_lut"] = [[float(v) for v in imgops.normalize(
        np.arange(256, dtype=np.uint8).reshape(16, 16, 1).repeat(3, 2))[c].ravel()]
        for c in range(3)]

    # ---- rng / sampling -----------------------------------------------------
    g["rng_u64"] = [str(R.SampleRng(5, 7, 11, d).next_u64()) for d in (0, 1, 3)]
    arrays["perm_3_2_1000"] = R.epoch_permutation(3, 2, 1000)
    arrays["perm_0_0_10"] = R.epoch_permutation(0, 0, 10)
    rc = RrcConfig()
    rects = []
    for (w, hgt) in ((256, 256), (500, 375), (20, 500), (512, 512), (1, 1), (300, 17)):
        for i in range(200):
            r = sample_rrc(R.SampleRng(1, 2, i), w, hgt, rc)
            rects.append([w, hgt, i, r.x, r.y, r.w, r.h])
    rc2 = RrcConfig(scale=(0.2, 1.0))
    for i in range(200):
        r = sample_rrc(R.SampleRng(9, 4, i), 512, 512, rc2)
        rects.append([512, 512, 10000 + i, r.x, r.y, r.w, r.h])
    arrays["rrc"] = np.array(rects, np.int64)
    masks = []
    for (res, m) in ((160, 0.5), (192, 0.66), (192, 0.8), (224, 0.75), (224, 0.85),
                     (112, 0.75), (224, 0.0), (224, 1.0)):
        spec = masking.MaskSpec.from_resolution(res, 16, m)
        for i in range(5):
            mk = masking.sample_mask(R.SampleRng(3, 1, i, R.DOMAIN_MASK), spec)
            masks.append({"res": res, "m": m, "i": i, "k": spec.masked_count,
                          "mask": mk.tolist()})
    g["masks"] = masks

    # ---- encoder (row f2 of SURVEY 8(f)) -------------------------------------
    enc_src = synth_image(31, 72, 104)
    arrays["encode_src"] = enc_src
    g["encode"] = {str(q): sha(encode_jpeg(enc_src, q)) for q in (50, 90, 95, 100)}
    g["encode_rst5"] = sha(encode_jpeg(enc_src, 90, restart_interval=5))

    (OUT / "golden.json").write_text(json.dumps(g, indent=1))
    np.savez_compressed(OUT / "arrays.npz", **arrays)
    print("wrote", OUT, file=sys.stderr)


if __name__ == "__main__":
    main()
