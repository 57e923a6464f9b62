"""multi-scan JPEG streams (progressive, and sequential
non-interleaved) decoded on the GPU exactly as the reference's full-decode
fallback (codec.py:352-399, 461-469; decode_kernels.py:111-385).  Goldens
come from the reference itself (tests/golden/make_golden_progressive.py):
full-image and crop SHA-256, DecodeStats (fallback_full set), the exact
error message and offset of damaged streams, and the reference Loader's
float32 pixels and masks over a container of progressive JPEGs."""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

GMS = json.loads((GOLDEN / "golden_ms.json").read_text())
NAMES = sorted(GMS["streams"])


def sha(a) -> str:
    if hasattr(a, "cpu"):
        a = a.cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def data_of(name: str) -> bytes:
    return (GOLDEN / "streams_ms" / f"{name}.jpg").read_bytes()


@pytest.fixture(scope="module")
def E(cuda):
    import paper_2404_00509_b200 as E
    return E


@pytest.mark.parametrize("name", NAMES)
def test_multiscan_stream_matches_reference(E, name):
    ent = GMS["streams"][name]
    data = data_of(name)
    if "error" in ent:
        with pytest.raises(E.DecodeError) as e:
            E.decode_full(data)
        assert str(e.value) == ent["error"]["msg"]
        return
    full, st = E.decode_full(data)
    assert sha(full) == ent["full"]["sha"]
    assert [st.mcus_entropy_decoded, st.mcus_reconstructed, st.fallback_full] == ent["full"]["stats"]
    items = [(data, E.CropRect(*c["rect"])) for c in ent["crops"]]
    for (crop, cs), c in zip(E.decode_crops(items), ent["crops"]):
        assert sha(crop) == c["sha"], c["rect"]
        assert [cs.mcus_entropy_decoded, cs.mcus_reconstructed, cs.fallback_full] == c["stats"]


def test_mixed_batch_baseline_and_multiscan(E, golden):
    """One batch mixing baseline and multi-scan streams (each image takes its
    own decode path inside the same launches)."""
    from conftest import stream_bytes
    items, exp = [], []
    for name in ("q92", "pil_444", "pil_gray"):
        for c in golden["streams"][name]["crops"][:4]:
            items.append((stream_bytes(name), E.CropRect(*c["rect"])))
            exp.append(c["sha"])
    for name in ("prog_420", "prog_gray", "seq_3scans", "prog_rst"):
        for c in GMS["streams"][name]["crops"][:4]:
            items.append((data_of(name), E.CropRect(*c["rect"])))
            exp.append(c["sha"])
    order = np.random.default_rng(0).permutation(len(items))
    got = E.decode_crops([items[i] for i in order])
    assert [sha(g[0]) for g in got] == [exp[i] for i in order]


@pytest.mark.parametrize("key", ["f32", "mask"])
def test_loader_over_progressive_container(E, key):
    """The Loader over a container of progressive / non-interleaved JPEGs ==
    the reference Loader, float32 pixels bit for bit, masks exact."""
    spec = GMS["loader"]
    kw = {"mask_ratio": 0.75} if key == "mask" else {}
    cfg = E.LoaderConfig(data=str(GOLDEN / "ms_small.essl"), batch_size=spec["batch"],
                         res=spec["res"], seed=spec["seed"], **kw)
    got = []
    with E.Loader(cfg) as loader:
        for b in loader.epoch(spec["epoch"]):
            for s in range(len(b)):
                got.append({"cfg": key, "index": int(b.indices[s]), "label": int(b.labels[s]),
                            "pixels": sha(b.pixels[s]),
                            "mask": b.mask[s].cpu().tolist() if b.mask is not None else None})
    assert got == [s for s in spec["samples"] if s["cfg"] == key]


GCL = json.loads((GOLDEN / "golden_clobber.json").read_text())


@pytest.mark.parametrize("name", sorted(GCL["streams"]))
def test_tables_read_before_the_inplace_destuff_clobbers_them(E, name):
    """Baseline streams whose last DHT ends right before SOS, scan start at
    15 mod 16: k_prep's in-place destuff overwrites the 15 bytes below the
    scan start (the SOS header and, for one component, the DHT's last 5
    symbols -- here frequent 8-bit codes).  The Huffman tables must come from
    the original bytes: decode_full and crops equal the reference's
    (tests/golden/make_golden_clobber.py); also decoded twice in one batch
    (the second copy hits the context's table cache)."""
    ent = GCL["streams"][name]
    data = (GOLDEN / "streams_clobber" / f"{name}.jpg").read_bytes()
    full, st = E.decode_full(data)
    assert sha(full) == ent["full"]["sha"]
    items = [(data, E.CropRect(*c["rect"])) for c in ent["crops"]] * 2
    for (crop, cs), c in zip(E.decode_crops(items), ent["crops"] * 2):
        assert sha(crop) == c["sha"], c["rect"]
        assert [cs.mcus_entropy_decoded, cs.mcus_reconstructed, cs.fallback_full] == c["stats"]
