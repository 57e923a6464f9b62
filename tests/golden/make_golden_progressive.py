"""Golden fixtures for multi-scan JPEG streams: the
reference's full-decode fallback (codec.py:352-399, 461-469 with
decode_kernels.py:111-385) run on progressive and non-interleaved streams.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_progressive.py

Streams come from Pillow (progressive, with and without restart markers,
4:2:0 / 4:2:2 / 4:4:4 / gray, optimized tables) and from a small
non-interleaved baseline writer below (three sequential scans, one per
component, Annex K tables) fed with the reference decoder's own coefficients.
Damaged variants (truncations, byte flips) record the reference's exact
errors.  A small container of progressive JPEGs records the reference
Loader's outputs.

Outputs (tests/golden/): streams_ms/*.jpg, golden_ms.json, ms_small.essl
"""

from __future__ import annotations

import hashlib
import io
import json
import zlib
from pathlib import Path

import numpy as np
from PIL import Image

from cropload.container import open_container
from cropload.errors import CroploadError
from cropload.jpeg import CropRect, decode_crop, decode_full
from cropload.jpeg import codec as C
from cropload.jpeg import tables as T
from cropload.pipeline import Loader, LoaderConfig
from cropload.synth import synth_image

OUT = Path(__file__).resolve().parent
SDIR = OUT / "streams_ms"


def sha(a) -> str:
    if isinstance(a, (bytes, bytearray)):
        return hashlib.sha256(a).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def pil_jpeg(img, **kw) -> bytes:
    buf = io.BytesIO()
    Image.fromarray(img).save(buf, "JPEG", **kw)
    return buf.getvalue()


# ---- non-interleaved baseline writer (one scan per component) --------------
class _Bits:
    def __init__(self):
        self.out = bytearray()
        self.acc = 0
        self.n = 0

    def put(self, v, k):
        for i in range(k - 1, -1, -1):
            self.acc = (self.acc << 1) | ((v >> i) & 1)
            self.n += 1
            if self.n == 8:
                self.out.append(self.acc)
                if self.acc == 0xFF:
                    self.out.append(0)
                self.acc = 0
                self.n = 0

    def flush(self):
        if self.n:
            self.put((1 << (8 - self.n)) - 1, 8 - self.n)
        return bytes(self.out)


def _codes(bits, vals):
    code, k, out = 0, 0, {}
    for L in range(1, 17):
        for _ in range(bits[L - 1]):
            out[vals[k]] = (code, L)
            code += 1
            k += 1
        code <<= 1
    return out


def _mag(v):
    a = abs(v)
    s = a.bit_length()
    return s, (v if v >= 0 else v + (1 << s) - 1)


def non_interleaved(data: bytes) -> bytes:
    """Re-encode a baseline stream's coefficients as three sequential scans."""
    frame = C.parse_stream(data)
    coefs = C._alloc_coefs(frame)
    C._decode_scans_full(frame, np.frombuffer(data, np.uint8), coefs)
    nat = np.array(T.ZIGZAG_TO_NATURAL)
    tabs = [T.huff_spec(T.HUFF_DC_LUMA) + T.huff_spec(T.HUFF_AC_LUMA),
            T.huff_spec(T.HUFF_DC_CHROMA) + T.huff_spec(T.HUFF_AC_CHROMA)]
    # header up to (excluding) the first SOS, then our DHTs and scans
    sos = data.index(b"\xff\xda")
    out = bytearray(data[:sos])
    for tc, th, bits, vals in ((0, 0, tabs[0][0], tabs[0][1]), (1, 0, tabs[0][2], tabs[0][3]),
                               (0, 1, tabs[1][0], tabs[1][1]), (1, 1, tabs[1][2], tabs[1][3])):
        body = bytes([tc << 4 | th]) + bytes(bits) + bytes(vals)
        out += b"\xff\xc4" + (len(body) + 2).to_bytes(2, "big") + body
    for ci, comp in enumerate(frame.comps):
        t = 0 if ci == 0 else 1
        dcc = _codes(tabs[t][0], tabs[t][1])
        acc = _codes(tabs[t][2], tabs[t][3])
        body = bytes([1, comp.cid, t << 4 | t, 0, 63, 0])
        out += b"\xff\xda" + (len(body) + 2).to_bytes(2, "big") + body
        bw = _Bits()
        pred = 0
        cf = coefs[ci]
        for by in range(comp.bh):
            for bx in range(comp.bw):
                blk = cf[by, bx][nat]
                d = int(blk[0]) - pred
                pred = int(blk[0])
                s, m = _mag(d)
                bw.put(*dcc[s])
                bw.put(m, s)
                run = 0
                last = max([k for k in range(1, 64) if blk[k] != 0], default=0)
                for k in range(1, last + 1):
                    v = int(blk[k])
                    if v == 0:
                        run += 1
                        continue
                    while run > 15:
                        bw.put(*acc[0xF0])
                        run -= 16
                    s, m = _mag(v)
                    bw.put(*acc[(run << 4) | s])
                    bw.put(m, s)
                    run = 0
                if last < 63:
                    bw.put(*acc[0x00])
        out += bw.flush()
    out += b"\xff\xd9"
    return bytes(out)


def record(data: bytes, rr) -> dict:
    ent = {"sha": sha(data), "crops": []}
    try:
        full, st = decode_full(data)
        ent["full"] = {"sha": sha(full), "shape": list(full.shape),
                       "stats": [st.mcus_entropy_decoded, st.mcus_reconstructed, bool(st.fallback_full)]}
        hgt, wid = full.shape[:2]
        rects = [(0, 0, wid, hgt)]
        for _ in range(10):
            cw = int(rr.integers(1, wid + 1)); ch = int(rr.integers(1, hgt + 1))
            rects.append((int(rr.integers(0, wid - cw + 1)), int(rr.integers(0, hgt - ch + 1)), cw, ch))
        for (x, y, cw, ch) in rects:
            crop, cs = decode_crop(data, CropRect(x, y, cw, ch))
            ent["crops"].append({"rect": [x, y, cw, ch], "sha": sha(crop),
                                 "stats": [cs.mcus_entropy_decoded, cs.mcus_reconstructed,
                                           bool(cs.fallback_full)]})
    except CroploadError as exc:
        ent["error"] = {"type": type(exc).__name__, "msg": str(exc),
                        "offset": getattr(exc, "offset", None)}
    return ent


def write_ms_container(path: Path, n: int = 24) -> None:
    """Reference-layout container (container.py:137-189, written by this
    repo's byte-identical writer) of progressive / multi-scan JPEGs."""
    import sys
    sys.path.insert(0, str(OUT.parent.parent))
    from paper_2404_00509_b200.container import write_container
    pays, ws, hs = [], [], []
    for i in range(n):
        h, w = 64 + 16 * (i % 4), 80 + 8 * (i % 5)
        im = synth_image(100 + i, h, w)
        if i % 6 == 5:
            pays.append(non_interleaved(pil_jpeg(im, quality=85)))
        else:
            pays.append(pil_jpeg(im, quality=80 + i % 15, progressive=True,
                                 subsampling=(2, 0, 1)[i % 3],
                                 **({"restart_marker_blocks": 2} if i % 4 == 3 else {})))
        ws.append(w)
        hs.append(h)
    write_container(path, pays, ws, hs, np.arange(n) % 5, 128, 85, 3)


def main():
    SDIR.mkdir(exist_ok=True)
    streams = {}
    img = synth_image(11, 180, 140)
    img2 = synth_image(12, 150, 200)
    streams["prog_420"] = pil_jpeg(img, quality=90, progressive=True)
    streams["prog_444"] = pil_jpeg(img2, quality=85, progressive=True, subsampling=0)
    streams["prog_422"] = pil_jpeg(img2, quality=85, progressive=True, subsampling=1)
    streams["prog_gray"] = pil_jpeg(np.asarray(Image.fromarray(img2).convert("L")), quality=88,
                                    progressive=True)
    streams["prog_opt"] = pil_jpeg(img, quality=75, progressive=True, optimize=True)
    streams["prog_odd"] = pil_jpeg(synth_image(13, 37, 61), quality=70, progressive=True)
    streams["prog_q100"] = pil_jpeg(synth_image(14, 96, 128), quality=100, progressive=True)
    streams["prog_big"] = pil_jpeg(synth_image(15, 256, 320), quality=95, progressive=True)
    streams["prog_rst"] = pil_jpeg(img2, quality=90, progressive=True, restart_marker_blocks=3)
    streams["prog_rst_rows"] = pil_jpeg(img, quality=80, progressive=True, restart_marker_rows=1)
    base = pil_jpeg(img2, quality=88, subsampling=2)
    streams["seq_3scans"] = non_interleaved(base)
    streams["seq_3scans_444"] = non_interleaved(pil_jpeg(img, quality=80, subsampling=0))
    # damaged streams: the reference's exact errors
    p = streams["prog_420"]
    for frac in (0.2, 0.45, 0.7, 0.93):
        streams[f"prog_cut_{int(frac * 100)}"] = p[:int(len(p) * frac)]
    r2 = np.random.default_rng(5)
    sos = p.index(b"\xff\xda")
    for i in range(6):
        b = bytearray(p)
        pos = int(r2.integers(sos + 20, len(b) - 4))
        b[pos] ^= int(r2.integers(1, 256))
        streams[f"prog_flip_{i}"] = bytes(b)
    g = {"streams": {}}
    for nm, data in streams.items():
        (SDIR / f"{nm}.jpg").write_bytes(data)
        g["streams"][nm] = record(data, np.random.default_rng(zlib.crc32(nm.encode())))
    # a small container of progressive JPEGs through the reference Loader
    path = OUT / "ms_small.essl"
    write_ms_container(path)
    samples = []
    for key, kw in (("f32", {}), ("mask", {"mask_ratio": 0.75})):
        cfg = LoaderConfig(data=str(path), batch_size=8, res=96, seed=3, workers=1, **kw)
        with Loader(cfg) as loader:
            for b in loader.epoch(1):
                for s in range(len(b.labels)):
                    samples.append({"cfg": key, "index": int(b.indices[s]), "label": int(b.labels[s]),
                                    "pixels": sha(b.pixels[s]),
                                    "mask": b.mask[s].tolist() if b.mask is not None else None})
    g["loader"] = {"res": 96, "seed": 3, "epoch": 1, "batch": 8, "samples": samples}
    (OUT / "golden_ms.json").write_text(json.dumps(g, indent=1))
    print(f"{len(streams)} streams, {len(samples)} loader samples")


if __name__ == "__main__":
    import sys
    sys.path.insert(0, str(OUT))
    main()
