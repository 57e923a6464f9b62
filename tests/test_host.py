"""Host-side product logic (no GPU): native sampling, encoder, container
format, schedules, config validation, DDP sharding."""

from __future__ import annotations

import hashlib
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT


def sha(b) -> str:
    return hashlib.sha256(b if isinstance(b, bytes) else np.ascontiguousarray(b).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def E(native):
    import paper_2404_00509_b200 as E
    return E


def test_native_exports_every_declared_symbol(native):
    """libessl.so loads without a GPU and exports every function essl.h declares."""
    header = (ROOT / "include" / "essl.h").read_text()
    declared = set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(essl_\w+)\s*\(", header, re.M))
    assert declared == set(native.EXPORTS)
    L = native.lib()
    for name in declared:
        assert getattr(L, name) is not None
    assert b"sm_100a" in L.essl_version()
    # option defaults are readable without a device (the GPU tests restore them)
    assert native.option_default(native.ESSL_OPT_SEQ_BITS) == 3072
    assert native.option_default(native.ESSL_OPT_WARMUP_BITS) == 2560
    assert native.option_default(native.ESSL_OPT_DECODE_MODE) == native.ESSL_DECODE_SPECULATIVE


def test_abi_struct_sizes_match_ctypes(native):
    """The ctypes mirrors in _native.py have the C structs' sizes (a field
    added on one side only would shift every later field)."""
    import ctypes
    out = (ctypes.c_int64 * 5)()
    assert native.lib().essl_abi_sizes(ctypes.cast(out, ctypes.c_void_p), 5) == 5
    mine = [ctypes.sizeof(t) for t in (native.EsslSample, native.EsslResult, native.EsslAug,
                                       native.EsslBatchCfg, native.EsslBatchIo)]
    assert list(out) == mine


def test_rng_and_permutation(E, golden, arrays):
    assert [str(E.SampleRng(5, 7, 11, d).next_u64()) for d in (0, 1, 3)] == golden["rng_u64"]
    assert np.array_equal(E.epoch_permutation(3, 2, 1000), arrays["perm_3_2_1000"])
    r = E.SampleRng(1, 2, 3)
    vals = [r.randint(10) for _ in range(1000)]
    assert min(vals) == 0 and max(vals) == 9


def test_rrc_matches_reference_vectors(E, arrays):
    for w, h, i, x, y, cw, ch in arrays["rrc"]:
        if i >= 10000:
            cfg = E.RrcConfig(scale=(0.2, 1.0))
            r = E.sample_rrc(E.SampleRng(9, 4, int(i) - 10000), int(w), int(h), cfg)
        else:
            r = E.sample_rrc(E.SampleRng(1, 2, int(i)), int(w), int(h), E.RrcConfig())
        assert (r.x, r.y, r.w, r.h) == (x, y, cw, ch)


def test_rrc_batch_matches_loader_golden(E, golden, native):
    spec = golden["loader"]["cfg1_simple_224"]
    with E.open_container(GOLDEN / spec["data"]) as h:
        ws = np.ascontiguousarray(h.records["width"], np.uint16)
        hs = np.ascontiguousarray(h.records["height"], np.uint16)
        for e in (0, 1):
            smp = [s for s in spec["samples"] if s["epoch"] == e]
            idx = np.array([s["index"] for s in smp], np.int64)
            out = np.zeros(len(idx), native._np_dtypes()[0])
            native.check(native.lib().essl_rrc_batch(0, e, native.ptr(idx), len(idx),
                                                     native.ptr(ws), native.ptr(hs), 0.08, 1.0,
                                                     0.75, 4 / 3, native.ptr(out)))
            for o, s in zip(out, smp):
                assert [o["x"], o["y"], o["w"], o["h"]] == s["rect"] and o["flip"] == s["flip"]


def test_rrc_statistics(E):
    # test_pipeline.py:52-70: mean accepted area 0.4331 on 500x375
    cfg = E.RrcConfig()
    fr = []
    for i in range(20000):
        r = E.sample_rrc(E.SampleRng(123, 0, i), 500, 375, cfg)
        assert r.x >= 0 and r.y >= 0 and r.x + r.w <= 500 and r.y + r.h <= 375
        fr.append(r.w * r.h / (500 * 375))
    assert abs(np.mean(fr) - 0.4331) < 0.01


def test_mask_count(E, native):
    for res, m, k in ((160, .5, 50), (192, .66, 95), (192, .8, 115), (224, .75, 147),
                      (224, .85, 167)):
        assert E.MaskSpec.from_resolution(res, 16, m).masked_count == k
        assert native.lib().essl_mask_count((res // 16) ** 2, m) == k


def test_encoder_byte_identical_to_reference(E, golden, arrays):
    src = arrays["encode_src"]
    for q, digest in golden["encode"].items():
        assert sha(E.encode_jpeg(src, int(q))) == digest
    assert sha(E.encode_jpeg(src, 90, restart_interval=5)) == golden["encode_rst5"]
    with pytest.raises(ValueError):
        E.encode_jpeg(src, 0)
    with pytest.raises(ValueError):
        E.encode_jpeg(src, 101)


def test_synth_and_builder(E, tmp_path):
    a = E.synth_image(7, 64, 80)
    assert np.array_equal(a, E.synth_image(7, 64, 80))
    assert not np.array_equal(a, E.synth_image(8, 64, 80))
    info = E.build_synthetic(tmp_path / "s.essl", 6, 96, 90, classes=3, seed=2, workers=2)
    with E.open_container(tmp_path / "s.essl") as h:
        assert len(h) == 6
        for i in range(6):
            payload, w, hh, label = h.read_sample(i)
            assert (w, hh) == (96, 96) and label == i % 3
    info = E.build_synthetic(tmp_path / "a.essl", 4, 64, 90, seed=3, n_records=37)
    with E.open_container(tmp_path / "a.essl") as h:
        assert len(h) == 37
        assert h.records["payload_offset"][5] == h.records["payload_offset"][1]
        h.read_sample(36)


def test_write_container_reproduces_reference_bytes(E, golden):
    """Re-packing the golden container's payloads yields the same file."""
    src = GOLDEN / "cfg1_small.essl"
    with E.open_container(src) as h:
        pays = [h.read_sample(i)[0] for i in range(len(h))]
        recs = h.records.copy()
        hd = h.header
    out = GOLDEN.parent / "_tmp_repack.essl"
    try:
        E.write_container(out, pays, recs["width"], recs["height"], recs["label"],
                          hd.max_resolution, hd.quality, hd.build_seed)
        assert sha(out.read_bytes()) == golden["containers"]["cfg1_small.essl"]["file_sha"]
    finally:
        out.unlink(missing_ok=True)


def test_container_errors(E, tmp_path):
    p = tmp_path / "bad.essl"
    p.write_bytes(b"XXXX" + bytes(60))
    with pytest.raises(E.FormatError):
        E.open_container(p)
    good = (GOLDEN / "cfg1_small.essl").read_bytes()
    corrupt = bytearray(good)
    with E.open_container(GOLDEN / "cfg1_small.essl") as h:
        off = int(h.records["payload_offset"][3])
    corrupt[off + 700] ^= 0x55
    p2 = tmp_path / "corrupt.essl"
    p2.write_bytes(bytes(corrupt))
    assert E.verify_crcs(p2) == [3]
    with E.open_container(p2) as h:
        with pytest.raises(E.CorruptionError, match="sample 3: checksum mismatch"):
            h.read_sample(3)
        with pytest.raises(IndexError):
            h.read_sample(len(h))


def test_schedule(E, golden):
    s = E.load_scheme(golden["scheme_prog4"])
    assert [E.params_for_epoch(s, e, 4).resolution for e in range(4)] == [112, 160, 192, 224]
    s1 = E.builtin_scheme("pt_s1")
    assert s1.boundaries(800) == [240, 480, 800]
    p = E.params_for_epoch(s1, 799, 800)
    assert (p.resolution, p.masking_ratio, p.stage) == (224, 0.75, 2)
    assert E.load_scheme(E.emit_schedule(s1, 10)) == s1
    with pytest.raises(E.ConfigError):
        E.builtin_scheme("nope")


def test_loader_config_validation(E):
    with pytest.raises(E.ConfigError, match="patch"):
        E.LoaderConfig(data="x", res=100, mask_ratio=0.5, patch=16).validate()
    with pytest.raises(E.ConfigError):
        E.LoaderConfig(data="x", aug="bogus").validate()
    with pytest.raises(E.ConfigError, match="unknown"):
        E.LoaderConfig.from_document({"data": "x", "bogus_key": 1})
    with pytest.raises(E.ConfigError, match="data"):
        E.LoaderConfig.from_document({"batch_size": 4})
    c = E.LoaderConfig.from_document('{"data": "x", "scale": [0.2, 1.0], "out_dtype": "bfloat16"}')
    assert c.scale == (0.2, 1.0) and c.out_dtype == "bfloat16"
    # GPU keys of the launch-set grouping and the host-staged fill
    c = E.LoaderConfig.from_document({"data": "x", "group": 2, "fill_chain": 0})
    assert (c.group, c.fill_chain) == (2, 0)
    assert (E.LoaderConfig(data="x").group, E.LoaderConfig(data="x").fill_chain) == (1, 0)
    with pytest.raises(E.ConfigError, match="group"):
        E.LoaderConfig(data="x", group=0).validate()
    with pytest.raises(E.ConfigError, match="fill_chain"):
        E.LoaderConfig(data="x", fill_chain=-1).validate()


def test_shard_partition(E):
    from paper_2404_00509_b200.rng import shard_len
    perm = E.epoch_permutation(0, 3, 1003)
    parts = [E.shard(perm, r, 4, "stride") for r in range(4)]
    assert sorted(np.concatenate(parts).tolist()) == list(range(1003))
    assert [len(p) for p in parts] == [251, 251, 251, 250]
    # default "pad": equal shards (every rank the same batch count), the
    # permutation wrapped around -- DistributedSampler semantics
    padded = [E.shard(perm, r, 4) for r in range(4)]
    assert [len(p) for p in padded] == [251] * 4
    assert padded[3][:-1].tolist() == parts[3].tolist() and padded[3][-1] == perm[0]
    assert set(np.concatenate(padded).tolist()) == set(range(1003))
    dropped = [E.shard(perm, r, 4, "drop") for r in range(4)]
    assert [len(p) for p in dropped] == [250] * 4
    for mode, ps in (("stride", parts), ("pad", padded), ("drop", dropped)):
        assert [shard_len(1003, r, 4, mode) for r in range(4)] == [len(p) for p in ps]
    assert E.shard(perm, 0, 1).tolist() == perm.tolist()
    with pytest.raises(ValueError):
        E.shard(perm, 4, 4)
    with pytest.raises(ValueError):
        E.shard(perm, 0, 4, "bogus")


# ---- 3-Aug draws and blur taps ---------------------------

def _gaug():
    import json
    return json.loads((GOLDEN / "golden_aug.json").read_text())


def test_aug_draws_match_reference(E):
    """essl_aug_draw (host C++) reproduces apply_aug's draws (pipeline.py:85-101)."""
    from paper_2404_00509_b200 import augment
    for rec in _gaug()["apply_aug"]:
        r = E.SampleRng(rec["seed"], rec["epoch"], rec["index"])
        flip, a = augment.draw(r._state, rec["level"])
        assert flip == rec["flip"] and int(a["op"][0]) == rec["op"]
        if rec["sigma"] is not None:
            assert float(a["sigma"][0]).hex() == rec["sigma"]
            assert int(a["radius"][0]) == rec["radius"]
        if rec["jitter"] is not None:
            assert [float(v).hex() for v in a["factors"][0]] == rec["jitter"]
        else:
            assert int(a["jitter"][0]) == 0


def test_aug_batch_matches_loader_golden(E, native):
    """essl_aug_batch: rects, flips and aug draws of the reference Loader."""
    from paper_2404_00509_b200 import augment
    g = _gaug()
    for key, spec in g["loader"].items():
        cfg = spec["cfg"]
        with E.open_container(GOLDEN / spec["data"]) as h:
            ws = np.ascontiguousarray(h.records["width"], np.uint16)
            hs = np.ascontiguousarray(h.records["height"], np.uint16)
            for e in spec["epochs"]:
                smp = [s for s in spec["samples"] if s["epoch"] == e]
                idx = np.array([s["index"] for s in smp], np.int64)
                s = np.zeros(len(idx), native._np_dtypes()[0])
                a = augment.new_aug(len(idx))
                sc = cfg.get("scale", (0.08, 1.0))
                native.check(native.lib().essl_aug_batch(
                    cfg["seed"], e, native.ptr(idx), len(idx), native.ptr(ws), native.ptr(hs),
                    sc[0], sc[1], 3 / 4, 4 / 3, augment.level_code(cfg["aug"]), native.ptr(s),
                    native.ptr(a)))
                augment.fill_weights(a)
                for i, ref in enumerate(smp):
                    assert [int(s[f][i]) for f in "xywh"] == ref["rect"], key
                    assert int(s["flip"][i]) == ref["flip"] and int(a["op"][i]) == ref["op"]
                    if ref["sigma"] is not None:
                        assert float(a["sigma"][i]).hex() == ref["sigma"]
                        w = [float(v).hex() for v in a["weights"][i][:2 * ref["radius"] + 1]]
                        assert w == ref["weights"], key
                    if ref["jitter"] is not None:
                        assert [float(v).hex() for v in a["factors"][i]] == ref["jitter"]


def test_blur_weights_vectorised_equal_reference_expression(E):
    """fill_weights groups a batch by radius into one numpy expression; it
    must equal imgops.py:157-160 evaluated per sample, element for element."""
    from paper_2404_00509_b200 import augment
    rr = np.random.default_rng(9)
    n = 4000
    a = augment.new_aug(n)
    a["op"] = 2
    a["sigma"] = 0.1 + 1.9 * rr.random(n)
    a["sigma"][:4] = (0.1, 1.0 / 3.0, 2.0 - 2 ** -52, 4.0)
    a["radius"] = [augment.blur_radius(float(s)) for s in a["sigma"]]
    augment.fill_weights(a)
    for i in range(n):
        w = augment.blur_weights(float(a["sigma"][i]))
        assert np.array_equal(a["weights"][i][:len(w)], w)
        assert not a["weights"][i][len(w):].any()


def test_aug_config_levels(E):
    from paper_2404_00509_b200 import augment
    assert augment.level_code("simple") == 0 and augment.level_code("3aug+") == 2
    with pytest.raises(ValueError):
        augment.level_code("4aug")
    with pytest.raises(E.ConfigError):
        E.LoaderConfig(data="x", aug="bogus").validate()
