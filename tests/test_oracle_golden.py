"""Pin the CPU oracle (oracle/essl_oracle.c) to the reference's own outputs.

The golden vectors were produced by the reference implementation itself
(tests/golden/make_golden.py); the oracle must reproduce every one of them
before it is trusted as the checker of the CUDA path.
"""

from __future__ import annotations

import hashlib
import zlib

import numpy as np
import pytest

from conftest import GOLDEN, stream_bytes


def sha(a) -> str:
    if isinstance(a, (bytes, bytearray)):
        return hashlib.sha256(a).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_rng_vectors(oracle, golden):
    got = [str(oracle.SampleRng(5, 7, 11, d).next_u64()) for d in (0, 1, 3)]
    assert got == golden["rng_u64"]


def test_epoch_permutation(oracle, arrays):
    assert np.array_equal(oracle.epoch_permutation(3, 2, 1000), arrays["perm_3_2_1000"])
    assert np.array_equal(oracle.epoch_permutation(0, 0, 10), arrays["perm_0_0_10"])


def test_rrc_vectors(oracle, arrays):
    for w, h, i, x, y, cw, ch in arrays["rrc"]:
        if i >= 10000:
            r = oracle.sample_rrc(oracle.SampleRng(9, 4, int(i) - 10000), int(w), int(h),
                                  scale=(0.2, 1.0))
        else:
            r = oracle.sample_rrc(oracle.SampleRng(1, 2, int(i)), int(w), int(h))
        assert r == (x, y, cw, ch)


def test_mask_vectors(oracle, golden):
    for m in golden["masks"]:
        grid = m["res"] // 16
        k = oracle.mask_count(grid * grid, m["m"])
        assert k == m["k"]
        got = oracle.sample_mask(oracle.SampleRng(3, 1, m["i"], 1), grid * grid, k)
        assert got.tolist() == m["mask"]


def test_mask_counts_published_pairs(oracle):
    # test_masking.py:13-23
    for res, m, k in ((160, .5, 50), (160, .75, 75), (192, .66, 95), (192, .75, 108),
                      (192, .8, 115), (224, .75, 147), (224, .85, 167)):
        assert oracle.mask_count((res // 16) ** 2, m) == k


def test_crc32_matches_zlib(oracle):
    rng = np.random.default_rng(0)
    for n in (0, 1, 3, 4, 5, 100, 4096, 28731):
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert oracle.crc32(b) == zlib.crc32(b)


def test_destuff_known_answer(oracle):
    # test_bench.py:139-148
    o, nr, end, clean, rst = oracle.destuff(b"\x01\xff\x00\x02\xff\xd0\x03\xff\xd9", 4)
    assert (o, nr, end) == (4, 1, 7)
    assert clean == b"\x01\xff\x02\x03"
    assert list(rst) == [3]


def test_idct_matches_reference_fixture(oracle, arrays, golden):
    # the full-stream crop hashes below exercise IDCT; this pins the
    # DC-only / zero paths on synthetic blocks too
    q = np.arange(1, 65, dtype=np.int32)
    flat = np.zeros(64, np.int32)
    flat[0] = 16
    blk = oracle.idct_block(flat, q)
    assert (blk == blk[0, 0]).all()


@pytest.mark.parametrize("name", ["q85_rst7", "q85_rst1", "q92", "q100", "q50_odd",
                                  "white_1x1", "flat_64", "pil_444", "pil_422", "pil_420_opt",
                                  "pil_gray"])
def test_stream_crops(oracle, golden, name):
    ent = golden["streams"][name]
    data = stream_bytes(name)
    full, st = oracle.decode_full(data)
    assert sha(full) == ent["full"]["sha"]
    assert list(st) == ent["full"]["stats"][:2]
    for c in ent["crops"]:
        crop, cs = oracle.decode_crop(data, tuple(c["rect"]))
        assert sha(crop) == c["sha"], c["rect"]
        assert list(cs) == c["stats"][:2]
        coefs = oracle.dump_coefs(data, tuple(c["rect"]))
        assert [sha(a) for a in coefs] == c["coef_sha"]
    for br in ent["bad_rects"]:
        with pytest.raises(oracle.OracleError) as e:
            oracle.decode_crop(data, tuple(br))
        assert e.value.status == oracle.ST_RECT


@pytest.mark.parametrize("name", ["truncated_half", "truncated_hdr", "not_jpeg"])
def test_stream_errors(oracle, golden, name):
    """Malformed streams: same exception type, message and byte offset as
    the reference (status -> message mapping of errors.status_error)."""
    from paper_2404_00509_b200.errors import status_error
    ent = golden["streams"][name]["error"]
    with pytest.raises(oracle.OracleError) as e:
        oracle.decode_full(stream_bytes(name))
    exc = status_error(e.value.status, e.value.reason, e.value.offset)
    assert type(exc).__name__ == ent["type"]
    assert str(exc) == ent["msg"]


def test_progressive_is_unsupported(oracle, golden):
    # the reference falls back to a full CPU decode (codec.py:461-469); the
    # GPU path (and therefore this oracle) reports "unsupported"
    assert golden["streams"]["pil_progressive"]["full"]["stats"][2] is False
    with pytest.raises(oracle.OracleError) as e:
        oracle.decode_full(stream_bytes("pil_progressive"))
    assert e.value.status == oracle.ST_UNSUPPORTED


def test_resize_vectors(oracle, golden, arrays):
    for i, r in enumerate(golden["resize"]):
        out = oracle.resize_bilinear(arrays[f"resize_src_{i}"], *r["out"])
        assert sha(out) == r["sha"]
    src = np.zeros((2, 2, 3), np.uint8)
    src[:, 1] = 255
    assert oracle.resize_bilinear(src, 4)[0, :, 0].tolist() == golden["resize_2x2_row"]


def test_normalize_vectors(oracle, golden, arrays):
    assert sha(oracle.normalize(arrays["normalize_src"])) == golden["normalize_sha"]
    lut = oracle.normalize(np.arange(256, dtype=np.uint8).reshape(16, 16, 1).repeat(3, 2))
    for c in range(3):
        assert lut[c].ravel().tolist() == golden["normalize_lut"][c]


def _records(path):
    from paper_2404_00509_b200.container import open_container
    return open_container(path)


@pytest.mark.parametrize("key", ["cfg1_simple_224", "cfg1_mask_224", "cfg4_pt_224",
                                 "mixed_96_u8", "cfg3_epoch0", "cfg3_epoch1", "cfg3_epoch2",
                                 "cfg3_epoch3"])
def test_loader_end_to_end(oracle, golden, key):
    spec = golden["loader"][key]
    cfg = spec["cfg"]
    with _records(GOLDEN / spec["data"]) as h:
        for s in spec["samples"]:
            payload, w, hh, label = h.read_sample(s["index"])
            rec = h.records[s["index"]]
            pix, u8, mask, rect = oracle.fill_sample(
                payload, int(rec["checksum"]), w, hh, s["index"], cfg["seed"], s["epoch"],
                cfg["res"], scale=tuple(cfg.get("scale", (0.08, 1.0))),
                mask_ratio=cfg.get("mask_ratio", 0.0), patch=cfg.get("patch", 16))
            assert list(rect[:4]) == s["rect"] and rect[4] == s["flip"]
            assert sha(pix) == s["pixels"]
            if s["uint8"]:
                assert sha(u8) == s["uint8"]
            if s["mask"] is not None:
                assert mask.tolist() == s["mask"]
            assert label == s["label"]


def test_loader_batch_threads_match(oracle):
    """The threaded oracle batch (the bench CPU baseline) equals per-sample."""
    from paper_2404_00509_b200.container import open_container
    with open_container(GOLDEN / "cfg1_small.essl") as h:
        idx = np.arange(len(h))
        a, _, ma, st = oracle.loader_batch(h.bytes, h.records, idx, 0, 0, 224, nthreads=4,
                                           mask_ratio=0.75)
        b, _, mb, st2 = oracle.loader_batch(h.bytes, h.records, idx, 0, 0, 224, nthreads=1,
                                            mask_ratio=0.75)
        assert (st == 0).all() and (st2 == 0).all()
        assert np.array_equal(a, b) and np.array_equal(ma, mb)


GCL = __import__("json").loads((GOLDEN / "golden_clobber.json").read_text())


@pytest.mark.parametrize("name", sorted(GCL["streams"]))
def test_clobber_window_streams(oracle, name):
    """Reference-decoded streams whose last DHT sits in the 16 bytes below a
    scan start at 15 mod 16 (tests/golden/make_golden_clobber.py)."""
    ent = GCL["streams"][name]
    data = (GOLDEN / "streams_clobber" / f"{name}.jpg").read_bytes()
    full, st = oracle.decode_full(data)
    assert sha(full) == ent["full"]["sha"]
    assert list(st) == ent["full"]["stats"][:2]
    for c in ent["crops"]:
        crop, cs = oracle.decode_crop(data, tuple(c["rect"]))
        assert sha(crop) == c["sha"], c["rect"]
