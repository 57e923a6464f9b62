"""CUDA path parity: every GPU output against the reference's golden vectors
and the pinned CPU oracle on identical inputs.  Bars (BASELINE.json
north_star): DCT coefficients, crop boxes, masks, ids bit-exact; uint8 and
float32 pixels bit-exact (stricter than +-1 LSB); bf16 within 1e-2 abs."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import GOLDEN, stream_bytes

pytestmark = pytest.mark.gpu

STREAMS = ["q85_rst7", "q85_rst1", "q92", "q100", "q50_odd", "white_1x1", "flat_64", "pil_444",
           "pil_422", "pil_420_opt", "pil_gray"]
BF16_TOL = 1e-2


def sha(a) -> str:
    if hasattr(a, "cpu"):
        import torch
        a = a.cpu()
        if a.dtype == torch.bfloat16:
            a = a.view(torch.int16)
        a = a.numpy()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def E(cuda):
    import paper_2404_00509_b200 as E
    return E


# speculative: library defaults; spec_dense: every lane on every stream, a
# checkpoint at every block start, no warm-up; spec_sparse: few, far-apart
# checkpoints (late merges, long continuations), the longest warm-up, and the
# clean stream read from global memory (no shared-memory staging);
# serial: one lane (validation mode).
MODES = {"speculative": (None, None, None, None), "spec_dense": (32, 1, 0, 65536),
         "spec_sparse": (64, 4096, 4096, 0), "serial": None}


@pytest.fixture(params=list(MODES))
def mode(request, E):
    from paper_2404_00509_b200 import _native as N
    from paper_2404_00509_b200.engine import default_engine
    eng = default_engine()
    m = MODES[request.param]
    eng.set_option(N.ESSL_OPT_DECODE_MODE, N.ESSL_DECODE_SERIAL if m is None else N.ESSL_DECODE_SPECULATIVE)
    if m and m[0]:
        eng.set_option(N.ESSL_OPT_SEQ_BITS, m[0])
        eng.set_option(N.ESSL_OPT_CHECKPOINT_BITS, m[1])
        eng.set_option(N.ESSL_OPT_WARMUP_BITS, m[2])
        eng.set_option(N.ESSL_OPT_STAGE_BYTES, m[3])
    yield request.param
    # back to the library's own defaults (the default engine is shared)
    for opt in (N.ESSL_OPT_DECODE_MODE, N.ESSL_OPT_SEQ_BITS, N.ESSL_OPT_CHECKPOINT_BITS,
                N.ESSL_OPT_WARMUP_BITS, N.ESSL_OPT_STAGE_BYTES):
        eng.set_option(opt, N.option_default(opt))


@pytest.mark.parametrize("name", STREAMS)
def test_stream_crops_match_reference(E, golden, name, mode):
    ent = golden["streams"][name]
    data = stream_bytes(name)
    full, st = E.decode_full(data)
    assert sha(full) == ent["full"]["sha"]
    assert [st.mcus_entropy_decoded, st.mcus_reconstructed] == ent["full"]["stats"][:2]
    items = [(data, E.CropRect(*c["rect"])) for c in ent["crops"]]
    for (crop, cs), c in zip(E.decode_crops(items), ent["crops"]):
        assert sha(crop) == c["sha"], c["rect"]
        assert [cs.mcus_entropy_decoded, cs.mcus_reconstructed] == c["stats"][:2]
    for br in ent["bad_rects"]:
        with pytest.raises(ValueError):
            E.decode_crop(data, E.CropRect(*br))


@pytest.mark.parametrize("name", STREAMS)
def test_coefficients_bit_exact(E, oracle, golden, name, mode):
    """int16 crop-window coefficients == the reference's int32 arrays."""
    import torch
    from paper_2404_00509_b200.engine import default_engine
    eng = default_engine()
    data = stream_bytes(name)
    for c in golden["streams"][name]["crops"][:6]:
        rect = c["rect"]
        ref = oracle.dump_coefs(data, tuple(rect))
        assert [hashlib.sha256(a.tobytes()).hexdigest() for a in ref] == c["coef_sha"]
        blob = torch.from_numpy(np.frombuffer(data + bytes(64), np.uint8).copy()).to(eng.device)
        s = eng.samples(1)
        s["length"] = len(data)
        s["x"], s["y"], s["w"], s["h"] = rect
        cap = sum(a.size for a in ref)
        out = torch.zeros(cap, dtype=torch.int16, device=eng.device)
        res = eng.new_results(1)
        geo = eng.dump_coefs(blob.data_ptr(), s, out, np.zeros(1, np.uint64), cap, res,
                             max_side=4096)
        assert res.cpu().numpy()[0, 0] == 0
        o = out.cpu().numpy()
        pos = 0
        for comp, a in enumerate(ref):
            by0, bx0, bh, bw = geo[0, comp]
            win = o[pos:pos + bh * bw * 64].reshape(bh, bw, 64)
            pos += bh * bw * 64
            assert np.array_equal(win, a[by0:by0 + bh, bx0:bx0 + bw]), (name, rect, comp)


@pytest.mark.parametrize("name", ["truncated_half", "truncated_hdr", "not_jpeg"])
def test_stream_errors_match_reference(E, golden, name, mode):
    ent = golden["streams"][name]["error"]
    with pytest.raises(E.DecodeError) as e:
        E.decode_full(stream_bytes(name))
    assert str(e.value) == ent["msg"]


def test_progressive_decodes_like_reference(E, golden, mode):
    """Multi-scan streams take the reference's full-decode path on the GPU
    (codec.py:461-469): crops and stats (fallback_full set) == the goldens."""
    ent = golden["streams"]["pil_progressive"]
    data = stream_bytes("pil_progressive")
    full, st = E.decode_full(data)
    assert sha(full) == ent["full"]["sha"]
    assert [st.mcus_entropy_decoded, st.mcus_reconstructed, st.fallback_full] == ent["full"]["stats"]
    items = [(data, E.CropRect(*c["rect"])) for c in ent["crops"]]
    for (crop, cs), c in zip(E.decode_crops(items), ent["crops"]):
        assert sha(crop) == c["sha"], c["rect"]
        assert [cs.mcus_entropy_decoded, cs.mcus_reconstructed, cs.fallback_full] == c["stats"]


def test_truncation_every_cut(E, oracle):
    """Cut a stream at many points: GPU status/offset == oracle (== ref)."""
    from paper_2404_00509_b200.errors import status_error
    data = stream_bytes("q92")
    rect = E.CropRect(0, 0, 64, 40)
    cuts = list(range(620, len(data), 997)) + [len(data) - 1, len(data) - 2]
    for cut in cuts:
        d = data[:cut]
        try:
            oracle.decode_crop(d, (rect.x, rect.y, rect.w, rect.h))
            ref = None
        except oracle.OracleError as e:
            ref = str(status_error(e.status, e.reason, e.offset))
        try:
            E.decode_crop(d, rect)
            got = None
        except Exception as e:  # noqa: BLE001
            got = str(e)
        assert got == ref, cut


def test_corruption_every_flip(E, oracle, mode):
    """Flip entropy-coded bytes at many points: GPU status/offset or pixels ==
    oracle (corrupt codes on the exact path, inside merges, near the end)."""
    from paper_2404_00509_b200.errors import status_error
    data = stream_bytes("q92")
    info = oracle.jpeg_info(data)
    for rect in ((0, 0, 64, 40), (0, 0, info["width"], info["height"])):
        for pos in range(info["scan_start"] + 3, info["scan_end"] - 1, 331):
            d = bytearray(data)
            d[pos] ^= 0x5A
            d = bytes(d)
            try:
                ref, ref_err = oracle.decode_crop(d, rect)[0], None
            except oracle.OracleError as e:
                ref, ref_err = None, str(status_error(e.status, e.reason, e.offset))
            try:
                got, got_err = E.decode_crop(d, E.CropRect(*rect))[0], None
            except Exception as e:  # noqa: BLE001
                got, got_err = None, str(e)
            assert got_err == ref_err, (pos, rect, mode)
            if ref is not None:
                assert np.array_equal(np.asarray(got.cpu() if hasattr(got, "cpu") else got), ref), (pos, rect, mode)


def _golden_loader(E, golden, key, dtype="float32"):
    spec = golden["loader"][key]
    cfg = dict(spec["cfg"])
    cfg.update(data=str(GOLDEN / spec["data"]), workers=2, out_dtype=dtype)
    return spec, E.Loader(E.LoaderConfig(**{k: (tuple(v) if isinstance(v, list) else v)
                                            for k, v in cfg.items()}))


@pytest.mark.parametrize("key", ["cfg1_simple_224", "cfg1_mask_224", "cfg4_pt_224",
                                 "mixed_96_u8", "cfg3_epoch0", "cfg3_epoch1", "cfg3_epoch2",
                                 "cfg3_epoch3"])
def test_loader_float32_bit_exact(E, golden, key):
    spec, loader = _golden_loader(E, golden, key)
    with loader:
        got = []
        for e in spec["epochs"]:
            for b in loader.epoch(e):
                for s in range(len(b)):
                    got.append((e, int(b.indices[s]), int(b.labels[s]), sha(b.pixels[s]),
                                sha(b.uint8[s]) if b.uint8 is not None else None,
                                b.mask[s].cpu().tolist() if b.mask is not None else None))
    exp = [(s["epoch"], s["index"], s["label"], s["pixels"], s["uint8"], s["mask"])
           for s in spec["samples"]]
    assert got == exp


def test_loader_bf16_within_tolerance(E, golden, oracle):
    import torch
    spec, loader = _golden_loader(E, golden, "cfg1_mask_224", dtype="bfloat16")
    _, loader32 = _golden_loader(E, golden, "cfg1_mask_224")
    with loader, loader32:
        for b16, b32 in zip(loader.epoch(0), loader32.epoch(0)):
            d = (b16.pixels.float() - b32.pixels).abs().max().item()
            assert d <= BF16_TOL
            assert torch.equal(b16.pixels, b32.pixels.to(torch.bfloat16))  # exact RNE
            # ids_keep / ids_restore are the MAE conventions over the mask
            T = b16.ids_restore.shape[1]
            for s in range(len(b16)):
                m = b16.mask[s].cpu().numpy()
                keep = np.setdiff1d(np.arange(T), m)
                assert np.array_equal(b16.ids_keep[s].cpu().numpy(), keep)
                shuffle = np.concatenate([keep, m])
                assert np.array_equal(b16.ids_restore[s].cpu().numpy(), np.argsort(shuffle))


def test_gather_visible(E, golden):
    import torch
    from paper_2404_00509_b200.engine import default_engine
    spec, loader = _golden_loader(E, golden, "cfg1_mask_224", dtype="bfloat16")
    with loader:
        b = next(iter(loader.epoch(0)))
    eng = default_engine()
    n, p, res = len(b), 16, 224
    keep = b.ids_keep.to(eng.device)
    tok = torch.empty((n, keep.shape[1], p * p * 3), dtype=torch.bfloat16, device=eng.device)
    eng.gather_visible(b.pixels.to(eng.device), res, p, keep, tok)
    x = b.pixels.to(eng.device).reshape(n, 3, res // p, p, res // p, p)
    patches = torch.einsum("nchpwq->nhwpqc", x).reshape(n, (res // p) ** 2, p * p * 3)
    ref = torch.gather(patches, 1, keep[:, :, None].expand(-1, -1, p * p * 3))
    assert torch.equal(tok, ref)


def test_standalone_imgops(E, golden, arrays):
    for i, r in enumerate(golden["resize"]):
        assert sha(E.imgops.resize_bilinear(arrays[f"resize_src_{i}"], *r["out"])) == r["sha"]
    src = np.zeros((2, 2, 3), np.uint8)
    src[:, 1] = 255
    assert E.imgops.resize_bilinear(src, 4)[0, :, 0].tolist() == golden["resize_2x2_row"]
    assert sha(E.imgops.normalize(arrays["normalize_src"])) == golden["normalize_sha"]


def test_sample_mask_matches_reference(E, golden):
    for m in golden["masks"]:
        spec = E.MaskSpec.from_resolution(m["res"], 16, m["m"])
        rng = E.SampleRng(3, 1, m["i"], E.DOMAIN_MASK)
        assert E.sample_mask(rng, spec).tolist() == m["mask"]


def test_crc_corruption_raises(E, tmp_path):
    good = bytearray((GOLDEN / "cfg1_small.essl").read_bytes())
    with E.open_container(GOLDEN / "cfg1_small.essl") as h:
        off = int(h.records["payload_offset"][5])
    good[off + 1000] ^= 0x21
    p = tmp_path / "c.essl"
    p.write_bytes(bytes(good))
    with E.Loader(E.LoaderConfig(data=str(p), batch_size=16, res=64)) as loader:
        with pytest.raises(E.CorruptionError, match="sample 5: checksum mismatch"):
            list(loader.epoch(0))


@pytest.fixture(scope="module")
def synth_sets(E, tmp_path_factory):
    d = tmp_path_factory.mktemp("synth")
    a = d / "s256.essl"
    E.build_synthetic(a, 96, 256, 95, seed=5)
    b = d / "s512.essl"
    E.build_synthetic(b, 24, 512, 90, seed=6)
    c = d / "mixed.essl"
    E.build_synthetic(c, 40, (17, 333), 80, seed=7)
    return a, b, c


@pytest.mark.parametrize("seq_bits,ck_bits,warm,stage", [(4096, 64, 2048, 65536), (32, 1, 0, 65536),
                                                         (4096, 256, 4096, 0), (300, 5000, 300, 0)])
def test_speculative_vs_oracle_at_scale(E, oracle, synth_sets, seq_bits, ck_bits, warm, stage):
    """Synthetic datasets (random crops, all rows) through the checkpoint-merge
    decoder with adversarial lane / checkpoint settings == the oracle, bit for bit."""
    from paper_2404_00509_b200 import _native as N
    for path, scale in zip(synth_sets, ((0.08, 1.0), (0.2, 1.0), (0.08, 1.0))):
        with E.open_container(path) as h:
            cfg = E.LoaderConfig(data=str(path), batch_size=32, res=160, scale=scale,
                                 mask_ratio=0.75, keep_uint8=True)
            loader = E.Loader(cfg, container=h)
            loader.set_option(N.ESSL_OPT_SEQ_BITS, seq_bits)
            loader.set_option(N.ESSL_OPT_CHECKPOINT_BITS, ck_bits)
            loader.set_option(N.ESSL_OPT_WARMUP_BITS, warm)
            loader.set_option(N.ESSL_OPT_STAGE_BYTES, stage)
            for b in loader.epoch(3):
                idx = b.indices.cpu().numpy()
                pix, u8, mask, st = oracle.loader_batch(h.bytes, h.records, idx, 0, 3, 160,
                                                        scale=scale, mask_ratio=0.75,
                                                        keep_uint8=True, nthreads=8)
                assert (st == 0).all()
                assert np.array_equal(b.pixels.cpu().numpy(), pix)
                assert np.array_equal(b.uint8.cpu().numpy(), u8)
                assert np.array_equal(b.mask.cpu().numpy(), mask)


@pytest.mark.parametrize("stage", [65536, 0])
def test_large_pool_vs_oracle(E, oracle, tmp_path, stage):
    """1024 images of 256px q95 in batches of 256 (the bench's shape): every
    image bit-exact against the oracle, through the read rings (stage) and
    the plain global reader (0)."""
    from paper_2404_00509_b200 import _native as N
    path = tmp_path / "pool.essl"
    E.build_synthetic(path, 1024, 256, 95, seed=3)
    cfg = E.LoaderConfig(data=str(path), batch_size=256, res=224, streams=1, prefetch=1)
    with E.open_container(path) as h:
        loader = E.Loader(cfg, container=h)
        loader.set_option(N.ESSL_OPT_STAGE_BYTES, stage)
        for b in loader.epoch(0):
            idx = b.indices.cpu().numpy()
            pix, _, _, st = oracle.loader_batch(h.bytes, h.records, idx, 0, 0, 224, nthreads=8)
            assert (st == 0).all()
            assert np.array_equal(b.pixels.cpu().numpy(), pix)


@pytest.mark.parametrize("gather", [(8, 0), (0, 0), (3, 1), (8, 1), (0, 1)])
def test_staged_equals_resident(E, synth_sets, gather):
    """Host-container paths (bus-read gather: LSU or bulk-copy variant, few
    or one-per-payload CTAs; host-thread copy) == the HBM-resident container."""
    from paper_2404_00509_b200 import _native as N
    outs = []
    for resident, staging in ((True, "gather"), (False, "gather"), (False, "copy")):
        cfg = E.LoaderConfig(data=str(synth_sets[2]), batch_size=40, res=224,
                             out_dtype="bfloat16", resident=resident, prefetch=3,
                             staging=staging)
        with E.Loader(cfg) as loader:
            loader.set_option(N.ESSL_OPT_GATHER_CTAS, gather[0])
            loader.set_option(N.ESSL_OPT_GATHER_TMA, gather[1])
            outs.append([sha(b.pixels) for b in loader.epoch(1)])
    assert outs[0] == outs[1] == outs[2]


def test_ddp_shards_cover_epoch(E, synth_sets):
    path = synth_sets[2]
    seen = {}
    for r in range(3):
        cfg = E.LoaderConfig(data=str(path), batch_size=7, res=64, rank=r, world_size=3,
                             shard_mode="stride")
        with E.Loader(cfg) as loader:
            for b in loader.epoch(2):
                for s in range(len(b)):
                    seen[int(b.indices[s])] = sha(b.pixels[s])
    cfg = E.LoaderConfig(data=str(path), batch_size=7, res=64)
    with E.Loader(cfg) as loader:
        full = {int(b.indices[s]): sha(b.pixels[s]) for b in loader.epoch(2) for s in range(len(b))}
    assert seen == full


def test_multi_epoch_iterator_equals_epochs(E, synth_sets):
    """Loader.epochs(first, count) keeps the pipeline full across epoch
    boundaries and yields exactly the batches of consecutive epoch() calls."""
    path = synth_sets[2]
    cfg = E.LoaderConfig(data=str(path), batch_size=16, res=96, out_dtype="bfloat16",
                         mask_ratio=0.75, prefetch=3, streams=3)
    with E.Loader(cfg) as loader:
        a = [(sha(b.pixels), sha(b.indices), sha(b.mask)) for e in (4, 5, 6)
             for b in loader.epoch(e)]
        b = [(sha(x.pixels), sha(x.indices), sha(x.mask)) for x in loader.epochs(4, 3)]
        c = []
        for x in loader.epochs(4):
            c.append((sha(x.pixels), sha(x.indices), sha(x.mask)))
            if len(c) == len(a):
                break
        d = [(sha(x.pixels), sha(x.indices), sha(x.mask)) for x in loader.epochs(4, steps=len(a) - 1)]
    assert a == b == c
    assert d == a[:-1]


@pytest.mark.parametrize("res", [97, 16, 300])
def test_odd_and_extreme_resolutions_vs_oracle(E, oracle, synth_sets, res):
    """Output sizes off the paired-store fast path (odd), tiny, and larger than
    the crop (upscale, > the CTA's column count): float32 and the uint8 view
    bit-exact, bf16 the RNE of the float32."""
    import torch
    path = synth_sets[2]
    with E.open_container(path) as h:
        cfg = E.LoaderConfig(data=str(path), batch_size=20, res=res, keep_uint8=True)
        cfg16 = E.LoaderConfig(data=str(path), batch_size=20, res=res, out_dtype="bfloat16")
        l32, l16 = E.Loader(cfg, container=h), E.Loader(cfg16, container=h)
        for b, b16 in zip(l32.epoch(5), l16.epoch(5)):
            idx = b.indices.cpu().numpy()
            pix, u8, _, st = oracle.loader_batch(h.bytes, h.records, idx, 0, 5, res,
                                                 keep_uint8=True, nthreads=8)
            assert (st == 0).all()
            assert np.array_equal(b.uint8.cpu().numpy(), u8)
            assert np.array_equal(b.pixels.cpu().numpy(), pix)
            assert torch.equal(b16.pixels, b.pixels.to(torch.bfloat16))


@pytest.mark.parametrize("side,res", [(112, 224), (448, 224), (224, 112), (96, 160)])
def test_resize_dyadic_weights_vs_oracle(E, oracle, tmp_path, side, res):
    """Whole-image crops with power-of-two scale factors: the bilinear weights
    are dyadic (0.25 / 0.5 / 0.75), so many float64 values land exactly on
    integers -- the cases k_resize's float32 evaluation cannot decide and
    recomputes in float64.  uint8 and float32 bit-exact vs the oracle."""
    path = tmp_path / f"dy{side}.essl"
    E.build_synthetic(path, 24, side, 95, seed=11)
    with E.open_container(path) as h:
        cfg = E.LoaderConfig(data=str(path), batch_size=24, res=res, scale=(1.0, 1.0),
                             ratio=(1.0, 1.0), keep_uint8=True)
        loader = E.Loader(cfg, container=h)
        for b in loader.epoch(0):
            idx = b.indices.cpu().numpy()
            pix, u8, _, st = oracle.loader_batch(h.bytes, h.records, idx, 0, 0, res,
                                                 scale=(1.0, 1.0), ratio=(1.0, 1.0),
                                                 keep_uint8=True, nthreads=8)
            assert (st == 0).all()
            assert np.array_equal(b.uint8.cpu().numpy(), u8)
            assert np.array_equal(b.pixels.cpu().numpy(), pix)


@pytest.mark.parametrize("res", [64, 160, 224])
def test_loader_sampling_layouts_vs_oracle(E, oracle, tmp_path, res):
    """Every fixture stream layout (4:2:0, 4:2:2, 4:4:4, gray, restart
    intervals, odd sizes, 1x1) packed in a container and run through the
    loader (k_resize's colour-conversion paths): uint8 and float32 bit-exact
    vs the oracle."""
    from PIL import Image
    import io
    names = [n for n in STREAMS] * 3
    pay = [stream_bytes(n) for n in names]
    dims = [Image.open(io.BytesIO(b)).size for b in pay]
    path = tmp_path / "layouts.essl"
    E.write_container(path, pay, [d[0] for d in dims], [d[1] for d in dims],
                      list(range(len(pay))), max_resolution=512, quality=95)
    with E.open_container(path) as h:
        cfg = E.LoaderConfig(data=str(path), batch_size=16, res=res, keep_uint8=True)
        loader = E.Loader(cfg, container=h)
        for b in loader.epoch(2):
            idx = b.indices.cpu().numpy()
            pix, u8, _, st = oracle.loader_batch(h.bytes, h.records, idx, 0, 2, res,
                                                 keep_uint8=True, nthreads=8)
            assert (st == 0).all()
            assert np.array_equal(b.uint8.cpu().numpy(), u8)
            assert np.array_equal(b.pixels.cpu().numpy(), pix)


def test_resize_large_crops_smaller_bands_vs_oracle(E, oracle, tmp_path):
    """Crops large enough that k_resize's 32-row bands do not fit the shared
    staging: the host falls back to smaller bands; bit-exact vs the oracle."""
    path = tmp_path / "large.essl"
    E.build_synthetic(path, 8, (800, 900), 90, seed=13)
    with E.open_container(path) as h:
        cfg = E.LoaderConfig(data=str(path), batch_size=8, res=224, scale=(0.9, 1.0),
                             keep_uint8=True)
        loader = E.Loader(cfg, container=h)
        for b in loader.epoch(1):
            idx = b.indices.cpu().numpy()
            pix, u8, _, st = oracle.loader_batch(h.bytes, h.records, idx, 0, 1, 224,
                                                 scale=(0.9, 1.0), keep_uint8=True, nthreads=8)
            assert (st == 0).all()
            assert np.array_equal(b.uint8.cpu().numpy(), u8)
            assert np.array_equal(b.pixels.cpu().numpy(), pix)


@pytest.mark.parametrize("ri", [1, 4, 16])
def test_restart_variant_loader_vs_oracle(E, oracle, tmp_path, ri):
    """The restart-marker container variant (DRI + RSTn every
    ri MCUs): restart intervals decode from exact entry states, one per lane;
    uint8 and float32 bit-exact vs the oracle."""
    path = tmp_path / f"rst{ri}.essl"
    E.build_synthetic(path, 24, (200, 300), 95, seed=17, restart_interval=ri)
    with E.open_container(path) as h:
        cfg = E.LoaderConfig(data=str(path), batch_size=12, res=160, keep_uint8=True,
                             mask_ratio=0.75)
        loader = E.Loader(cfg, container=h)
        for b in loader.epoch(4):
            idx = b.indices.cpu().numpy()
            pix, u8, mask, st = oracle.loader_batch(h.bytes, h.records, idx, 0, 4, 160,
                                                    mask_ratio=0.75, keep_uint8=True, nthreads=8)
            assert (st == 0).all()
            assert np.array_equal(b.uint8.cpu().numpy(), u8)
            assert np.array_equal(b.pixels.cpu().numpy(), pix)
            assert np.array_equal(b.mask.cpu().numpy(), mask)
