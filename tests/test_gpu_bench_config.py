"""Parity at the configurations the benchmark times.

bench.py times Loader(streams=8, prefetch=8, reuse_outputs=True, bf16, mask
0.75, resident, batch 256) over 256px q95 JPEGs; these tests run that exact
loader (plus the host-staged e2e variant, the fused visible tokens and
caller-owned output buffers) over >= 2048 images and check every batch
against the C oracle (oracle/essl_oracle.c, pinned to the reference's goldens):
pixels == RNE(oracle float32) (bf16, <= 1e-2 abs by construction), mask,
ids_keep and ids_restore exact.  Each batch is checked while the loader keeps
running ahead, and the previous batch is re-checked one step later (the
reference bindings' "valid until the next step" contract).
cfg4 (512px q90, RRC(0.2,1), batch 1024) and a cfg5-style aliasing container
(records >> distinct payloads, one partial epoch) get the same checks."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E(cuda):
    import paper_2404_00509_b200 as E
    return E


def _digest(t) -> str:
    import torch
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        t = t.view(torch.int16)
    return hashlib.sha256(t.contiguous().numpy().tobytes()).hexdigest()


def _check_batch(oracle, h, b, epoch, res, scale, mask_ratio, patch=16):
    import torch
    idx = b.indices.cpu().numpy()
    pix, _, mask, st = oracle.loader_batch(h.bytes, h.records, idx, 0, epoch, res, scale=scale,
                                           mask_ratio=mask_ratio, patch=patch)
    assert (st == 0).all()
    ref16 = torch.from_numpy(pix).to(torch.bfloat16)
    got = b.pixels.cpu()
    assert torch.equal(got, ref16), "pixels != RNE(oracle f32)"
    assert (got.float() - torch.from_numpy(pix)).abs().max().item() <= 1e-2
    assert np.array_equal(b.labels.cpu().numpy(), h.records["label"][idx].astype(np.int64))
    if mask_ratio > 0:
        T = (res // patch) ** 2
        m = b.mask.cpu().numpy()
        assert np.array_equal(m, mask)
        keep = np.stack([np.setdiff1d(np.arange(T), r) for r in m])
        assert np.array_equal(b.ids_keep.cpu().numpy(), keep)
        restore = np.stack([np.argsort(np.concatenate([k, r])) for k, r in zip(keep, m)])
        assert np.array_equal(b.ids_restore.cpu().numpy(), restore)
        if b.visible is not None:
            # patchify ('nchpwq->nhwpqc') of the normalized bf16 pixels at ids_keep
            g = res // patch
            x = ref16.reshape(len(idx), 3, g, patch, g, patch)
            tok = torch.einsum("nchpwq->nhwpqc", x).reshape(len(idx), g * g, patch * patch * 3)
            ref_vis = torch.gather(tok, 1, torch.from_numpy(keep)[:, :, None].expand(
                -1, -1, patch * patch * 3))
            assert torch.equal(b.visible.cpu(), ref_vis), "visible tokens != patchify[ids_keep]"
    return len(idx)


def _run(E, oracle, path, *, batch, res, scale, mask_ratio, epochs, resident=True,
         visible=False, into=False, max_batches=None, streams=8, group=1):
    import torch
    with E.open_container(path) as h:
        cfg = E.LoaderConfig(data=str(path), batch_size=batch, res=res, scale=scale,
                             mask_ratio=mask_ratio, out_dtype="bfloat16", resident=resident,
                             streams=streams, prefetch=streams, reuse_outputs=True,
                             visible=visible, group=group)
        loader = E.Loader(cfg, container=h)
        bufs = None
        if into:
            bufs = [torch.empty((batch, 3, res, res), dtype=torch.bfloat16, device="cuda")
                    for _ in range(streams + 2)]
        n = nb = 0
        prev = None
        for b in loader.epochs(epochs[0], len(epochs), into=bufs):
            if prev is not None:  # the previous batch is still intact one step later
                assert _digest(prev[0].pixels) == prev[1]
            e = int(b.epoch)
            n += _check_batch(oracle, h, b, e, res, scale, mask_ratio)
            if bufs is not None:
                assert b.pixels.data_ptr() == bufs[nb % len(bufs)].data_ptr()
            prev = (b, _digest(b.pixels))
            nb += 1
            if max_batches and nb >= max_batches:
                break
        loader.close()
    return n, nb


@pytest.fixture(scope="module")
def pool256(E, tmp_path_factory):
    path = tmp_path_factory.mktemp("bench") / "pool256.essl"
    E.build_synthetic(path, 2048, 256, 95, classes=1000, seed=1)
    return path


@pytest.mark.parametrize("group", [2, 1])
def test_bench_config_resident(E, oracle, pool256, group):
    """The exact timed configuration: 8 streams, prefetch 8, output ring,
    bf16 + mask 0.75, resident, batch 256, two batches per launch set
    (bench.py --group 2; and single batches); 2 epochs of 2048 images."""
    n, nb = _run(E, oracle, pool256, batch=256, res=224, scale=(0.08, 1.0), mask_ratio=0.75,
                 epochs=(0, 1), group=group)
    assert n == 4096 and nb == 16


def test_bench_config_host_staged(E, oracle, pool256):
    """The e2e leg: the same loader with the page-locked host container
    gathered over the bus each batch."""
    n, _ = _run(E, oracle, pool256, batch=256, res=224, scale=(0.08, 1.0), mask_ratio=0.75,
                epochs=(2,), resident=False, group=2)
    assert n == 2048


def test_launch_groups_partial_and_epoch_boundaries(E, oracle, pool256):
    """Groups of 3 batches over epochs of 10 2/3 batches of 192 (a partial
    last batch, groups cut at every epoch boundary), 3 streams: the same
    batches as single launches, each checked against the oracle."""
    n, nb = _run(E, oracle, pool256, batch=192, res=160, scale=(0.08, 1.0), mask_ratio=0.75,
                 epochs=(4, 5), streams=3, group=3)
    assert n == 4096 and nb == 22


def test_bench_config_visible_tokens_and_into(E, oracle, pool256):
    """Fused visible-token output and caller-owned pixel buffers at the
    bench configuration."""
    n, _ = _run(E, oracle, pool256, batch=256, res=224, scale=(0.08, 1.0), mask_ratio=0.75,
                epochs=(3,), visible=True, into=True)
    assert n == 2048


def test_cfg4_batch_1024(E, oracle, tmp_path):
    """cfg4: 1024 x 512px q90, RRC(0.2,1) -> 224, one batch of 1024."""
    path = tmp_path / "cfg4.essl"
    E.build_synthetic(path, 1024, 512, 90, classes=1000, seed=2)
    n, nb = _run(E, oracle, path, batch=1024, res=224, scale=(0.2, 1.0), mask_ratio=0.0,
                 epochs=(0, 1), streams=2)
    assert n == 2048 and nb == 2


def test_cfg5_aliasing_container(E, oracle, tmp_path):
    """cfg5-style container: 60,000 records aliasing 512 distinct payloads
    (offsets and CRCs per record), first 12 batches of an epoch."""
    path = tmp_path / "cfg5.essl"
    E.build_synthetic(path, 512, 256, 95, classes=1000, seed=4, n_records=60_000)
    n, nb = _run(E, oracle, path, batch=256, res=224, scale=(0.08, 1.0), mask_ratio=0.75,
                 epochs=(5,), max_batches=12)
    assert nb == 12 and n == 12 * 256


@pytest.mark.parametrize("res", [224, 112])
def test_visible_tokens_progressive(E, oracle, pool256, res):
    """Visible tokens at a progressive stage resolution (N = (res/16)^2)."""
    n, _ = _run(E, oracle, pool256, batch=64, res=res, scale=(0.08, 1.0), mask_ratio=0.75,
                epochs=(0,), visible=True, max_batches=4, streams=2)
    assert n == 256


def test_unstaged_resize_for_huge_crops(E, oracle, tmp_path):
    """A crop whose source rows exceed the resize kernel's shared-memory
    budget even at one output row per CTA (1024px crops at res 16) takes the
    unstaged path (planes read directly) and stays bit-exact."""
    path = tmp_path / "big.essl"
    E.build_synthetic(path, 6, 1024, 60, seed=9)
    with E.open_container(path) as h:
        for scale, res in (((1.0, 1.0), 16), ((0.9, 1.0), 20), ((0.08, 1.0), 224)):
            cfg = E.LoaderConfig(data=str(path), batch_size=6, res=res, scale=scale,
                                 keep_uint8=True, streams=1, prefetch=1)
            loader = E.Loader(cfg, container=h)
            for b in loader.epoch(0):
                idx = b.indices.cpu().numpy()
                pix, u8, _, st = oracle.loader_batch(h.bytes, h.records, idx, 0, 0, res,
                                                     scale=scale, keep_uint8=True)
                assert (st == 0).all()
                assert np.array_equal(b.pixels.cpu().numpy(), pix)
                assert np.array_equal(b.uint8.cpu().numpy(), u8)


@pytest.mark.parametrize("cols,band", [(8, 64), (4, 64), (2, 32), (8, 5), (4, 16), (2, 3), (8, 1)])
@pytest.mark.parametrize("res", [224, 97])
def test_resize_shapes_vs_oracle(E, oracle, tmp_path_factory, cols, band, res):
    """k_resize thread shapes (ESSL_OPT_RESIZE_COLS / _BAND: columns per
    thread, output rows per CTA; odd resolutions take the scalar stores)
    are all bit-exact in float32 and uint8."""
    from paper_2404_00509_b200 import _native as N
    path = tmp_path_factory.mktemp("rs") / "mixed.essl"
    E.build_synthetic(path, 48, (40, 300), 85, seed=11)
    with E.open_container(path) as h:
        cfg = E.LoaderConfig(data=str(path), batch_size=24, res=res, keep_uint8=True,
                             streams=1, prefetch=1)
        loader = E.Loader(cfg, container=h)
        loader.set_option(N.ESSL_OPT_RESIZE_COLS, cols)
        loader.set_option(N.ESSL_OPT_RESIZE_BAND, band)
        for b in loader.epoch(1):
            idx = b.indices.cpu().numpy()
            pix, u8, _, st = oracle.loader_batch(h.bytes, h.records, idx, 0, 1, res, keep_uint8=True)
            assert (st == 0).all()
            assert np.array_equal(b.pixels.cpu().numpy(), pix)
            assert np.array_equal(b.uint8.cpu().numpy(), u8)
        # the plain path (no uint8 view) too
        cfg2 = E.LoaderConfig(data=str(path), batch_size=24, res=res, streams=1, prefetch=1)
        loader2 = E.Loader(cfg2, container=h)
        loader2.set_option(N.ESSL_OPT_RESIZE_COLS, cols)
        loader2.set_option(N.ESSL_OPT_RESIZE_BAND, band)
        for b in loader2.epoch(2):
            idx = b.indices.cpu().numpy()
            pix, _, _, st = oracle.loader_batch(h.bytes, h.records, idx, 0, 2, res)
            assert np.array_equal(b.pixels.cpu().numpy(), pix)


def _skewed_container(E, path, n=24, side=256, seed=21):
    """Images whose entropy-coded bits sit in their bottom rows (flat top,
    noisy bottom quarter): the block-share estimate of where the crop's last
    needed row ends undershoots, so the N2 early exit must extend the path."""
    from paper_2404_00509_b200.container import encode_jpeg, write_container
    rng = np.random.default_rng(seed)
    pays = []
    for i in range(n):
        img = np.full((side, side, 3), 90 + i, np.uint8)
        cut = side * 3 // 4 - 8 * (i % 5)
        img[cut:] = rng.integers(0, 256, (side - cut, side, 3), dtype=np.uint8)
        pays.append(encode_jpeg(img, 95))
    write_container(path, pays, [side] * n, [side] * n, np.arange(n) % 4, side, 95, seed)
    return path


@pytest.mark.parametrize("kind", ["pool", "skewed"])
def test_early_exit_equals_full_decode(E, oracle, pool256, tmp_path, kind):
    """N2: the entropy decode stopping near the crop's last needed MCU row
    (ESSL_OPT_EARLY_EXIT, default on) gives the same pixels as decoding every
    bit, and both equal the oracle -- also on streams whose bits concentrate
    below the estimate (the serial extension of the last lane's path)."""
    import torch
    from paper_2404_00509_b200 import _native as N
    path = pool256 if kind == "pool" else _skewed_container(E, tmp_path / "skew.essl")
    with E.open_container(path) as h:
        outs = []
        for ee in (1, 0):
            cfg = E.LoaderConfig(data=str(path), batch_size=256 if kind == "pool" else 24, res=224,
                                 out_dtype="bfloat16", streams=2, prefetch=2)
            loader = E.Loader(cfg, container=h)
            loader.set_option(N.ESSL_OPT_EARLY_EXIT, ee)
            got = []
            for e in (0, 1):
                for b in loader.epoch(e):
                    idx = b.indices.cpu().numpy()
                    if ee == 1:
                        pix, _, _, st = oracle.loader_batch(h.bytes, h.records, idx, 0, e, 224)
                        assert (st == 0).all()
                        assert torch.equal(b.pixels.cpu(), torch.from_numpy(pix).to(torch.bfloat16))
                    got.append(_digest(b.pixels))
                    if kind == "pool" and len(got) >= 4:
                        break
            outs.append(got)
        assert outs[0] == outs[1]
