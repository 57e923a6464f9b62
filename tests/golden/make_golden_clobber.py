"""Golden fixtures for baseline streams whose last DHT ends right before the
SOS segment, with the scan start at offset 15 mod 16 (k_prep's in-place
destuff writes from the 16-byte boundary below the scan start, over the SOS
header and, for a 1-component scan, the last 5 bytes of that DHT).  The AC
tables give every used symbol an 8-bit code and list the most frequent ones
last, so a table rebuilt from overwritten bytes decodes differently.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_golden_clobber.py

Outputs (tests/golden/): streams_clobber/*.jpg, golden_clobber.json
(reference decode_full / decode_crop SHA-256 and stats, as golden_ms.json).
"""

from __future__ import annotations

import collections
import io
import json
import sys
from pathlib import Path

import numpy as np
from PIL import Image

from cropload.jpeg import codec as C
from cropload.jpeg import tables as T
from cropload.synth import synth_image

OUT = Path(__file__).resolve().parent
SDIR = OUT / "streams_clobber"
sys.path.insert(0, str(OUT))
from make_golden_progressive import _Bits, _codes, _mag, record  # noqa: E402


def _seg(marker: int, body: bytes) -> bytes:
    return bytes([0xFF, marker]) + (len(body) + 2).to_bytes(2, "big") + body


def _symbols(coefs_list, nat):
    """DC categories and AC (run << 4 | size) symbols the scan will code, with counts."""
    dc, ac = collections.Counter(), collections.Counter()
    for cf in coefs_list:
        pred = 0
        for by in range(cf.shape[0]):
            for bx in range(cf.shape[1]):
                blk = cf[by, bx][nat]
                d = int(blk[0]) - pred
                pred = int(blk[0])
                dc[_mag(d)[0]] += 1
                last = max([k for k in range(1, 64) if blk[k] != 0], default=0)
                run = 0
                for k in range(1, last + 1):
                    if blk[k] == 0:
                        run += 1
                        continue
                    while run > 15:
                        ac[0xF0] += 1
                        run -= 16
                    ac[(run << 4) | _mag(int(blk[k]))[0]] += 1
                    run = 0
                if last < 63:
                    ac[0x00] += 1
    return dc, ac


def _flat_table(counter, length=8):
    """Every used symbol at one code length, the most frequent listed last."""
    syms = [s for s, _ in sorted(counter.items(), key=lambda kv: kv[1])]
    assert len(syms) < (1 << length)
    bits = [0] * 16
    bits[length - 1] = len(syms)
    return bits, syms


def clobber_stream(img: np.ndarray, quality: int, gray: bool) -> bytes:
    buf = io.BytesIO()
    Image.fromarray(img if not gray else img[..., 0]).save(buf, "JPEG", quality=quality,
                                                         subsampling=0)
    data = buf.getvalue()
    frame = C.parse_stream(data)
    coefs = C._alloc_coefs(frame)
    C._decode_scans_full(frame, np.frombuffer(data, np.uint8), coefs)
    nat = np.array(T.ZIGZAG_TO_NATURAL)
    ncomp = len(frame.comps)
    # one DC and one AC table per component class (luma, chroma)
    groups = [[0]] + ([list(range(1, ncomp))] if ncomp > 1 else [])
    tabs = []
    for g in groups:
        dc, ac = _symbols([coefs[c] for c in g], nat)
        tabs.append((_flat_table(dc, 4 if len(dc) < 16 else 5), _flat_table(ac)))
    sof = data.index(b"\xff\xc0")
    dqt_end = sof  # SOI + APP0 + DQT(s) precede SOF0 in Pillow's output
    head = data[2:dqt_end]
    sof_seg = data[sof:sof + 2 + int.from_bytes(data[sof + 2:sof + 4], "big")]
    dhts = b""
    # the AC table of the last class goes last, right before SOS
    order = [(0, i) for i in range(len(tabs))] + [(1, i) for i in range(len(tabs))]
    for tc, th in order:
        bits, syms = tabs[th][tc]
        dhts += _seg(0xC4, bytes([tc << 4 | th]) + bytes(bits) + bytes(syms))
    sos_body = bytes([ncomp]) + b"".join(bytes([frame.comps[c].cid, (0 if c == 0 else 1) * 0x11])
                                         for c in range(ncomp)) + bytes([0, 63, 0])
    sos = _seg(0xDA, sos_body)
    # a COM segment pads the header so that the scan starts at 15 mod 16
    base = 2 + len(head) + len(sof_seg) + len(dhts) + len(sos)
    pad = (15 - (base + 4)) % 16
    com = _seg(0xFE, b"x" * pad)
    assert (base + len(com)) % 16 == 15
    # the scan: interleaved MCUs (1x1 sampling), this stream's own tables
    codes = [(_codes(*t[0]), _codes(*t[1])) for t in tabs]
    bw = _Bits()
    preds = [0] * ncomp
    cbh, cbw = coefs[0].shape[0], coefs[0].shape[1]
    for by in range(cbh):
        for bx in range(cbw):
            for c in range(ncomp):
                dcc, acc = codes[0 if c == 0 else 1]
                blk = coefs[c][by, bx][nat]
                d = int(blk[0]) - preds[c]
                preds[c] = int(blk[0])
                s, m = _mag(d)
                bw.put(*dcc[s])
                bw.put(m, s)
                last = max([k for k in range(1, 64) if blk[k] != 0], default=0)
                run = 0
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
    return b"\xff\xd8" + com + head + sof_seg + dhts + sos + bw.flush() + b"\xff\xd9"


def main():
    SDIR.mkdir(exist_ok=True)
    streams = {
        "gray_flat8": clobber_stream(synth_image(21, 64, 80), 90, gray=True),
        "gray_flat8_big": clobber_stream(synth_image(22, 128, 96), 75, gray=True),
        "color444_flat8": clobber_stream(synth_image(23, 72, 56), 85, gray=False),
    }
    g = {"streams": {}}
    for nm, data in streams.items():
        (SDIR / f"{nm}.jpg").write_bytes(data)
        scan_start = data.index(b"\xff\xda") + 2 + int.from_bytes(data[data.index(b"\xff\xda") + 2:][:2], "big")
        assert scan_start % 16 == 15, (nm, scan_start)
        g["streams"][nm] = record(data, np.random.default_rng(len(nm)))
        g["streams"][nm]["scan_start"] = scan_start
    (OUT / "golden_clobber.json").write_text(json.dumps(g, indent=1))
    print(json.dumps({k: ("error" in v, v.get("scan_start")) for k, v in g["streams"].items()}))


if __name__ == "__main__":
    main()
