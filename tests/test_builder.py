"""Dataset ingestion (container.py:91-189): source-tree
scan semantics on the CPU; the whole build (Pillow decode + EXIF, GPU
fit_to_resolution, native encoder, container layout) byte-identical to the
reference's build_container over the same tree (tests/golden/make_golden_build.py)."""

from __future__ import annotations

import hashlib
import json

import pytest

from conftest import GOLDEN

GB = json.loads((GOLDEN / "golden_build.json").read_text())


def test_scan_source_tree_semantics(tmp_path):
    import paper_2404_00509_b200 as E
    files, classes = E.scan_source_tree(GOLDEN / "build_src")
    assert classes == ["ant", "bee", "cat"]
    assert [(f.parent.name + "/" + f.name, lab) for f, lab in files] == [
        ("ant/a0.png", 0), ("ant/a1.jpg", 0), ("ant/a2.bmp", 0), ("bee/b0.png", 1),
        ("bee/b1.jpg", 1), ("cat/c0.png", 2), ("cat/c1.jpg", 2)]
    with pytest.raises(E.CroploadError, match="source directory not found"):
        E.scan_source_tree(tmp_path / "missing")
    with pytest.raises(E.CroploadError, match="no class subfolders"):
        E.scan_source_tree(tmp_path)
    (tmp_path / "x").mkdir()
    with pytest.raises(E.CroploadError, match="no images found"):
        E.scan_source_tree(tmp_path)
    with pytest.raises(ValueError):
        E.BuildSpec(tmp_path, 32, 90)
    from paper_2404_00509_b200.builder import fit_size
    assert fit_size(200, 130, 96) == (96, int(130 * 96 / 200 + 0.5))
    assert fit_size(77, 181, 96) == (int(77 * 96 / 181 + 0.5), 96)
    assert fit_size(40, 70, 96) == (40, 70)


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(GB["builds"])))
def test_build_container_byte_identical(tmp_path, cuda, i):
    import paper_2404_00509_b200 as E
    g = GB["builds"][i]
    out = tmp_path / "c.essl"
    s = E.build_container(E.BuildSpec(GOLDEN / "build_src", g["max_resolution"], g["quality"],
                                      g["seed"]), out, workers=3)
    assert (s.sample_count, s.total_bytes) == (g["samples"], g["total_bytes"])
    assert hashlib.sha256(out.read_bytes()).hexdigest() == g["sha256"]
    with E.open_container(out) as h:  # and it loads through the GPU loader
        with E.Loader(E.LoaderConfig(data=str(out), batch_size=7, res=64), container=h) as ld:
            assert len(next(iter(ld.epoch(0)))) == 7
