"""Golden for dataset ingestion (f2): a small class-subfolder source tree
(PNG / JPEG / BMP sources, some above max_resolution, one with an EXIF
orientation tag) and the reference's build_container output over it.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_build.py
"""
import hashlib
import json
from pathlib import Path

import numpy as np
from PIL import Image

from cropload.container import BuildSpec, build_container
from cropload.synth import synth_image

OUT = Path(__file__).resolve().parent
SRC = OUT / "build_src"


def main():
    rng = np.random.default_rng(7)
    for cls in ("ant", "bee", "cat"):
        (SRC / cls).mkdir(parents=True, exist_ok=True)
    items = [("ant/a0.png", 90, 120), ("ant/a1.jpg", 150, 96), ("ant/a2.bmp", 40, 70),
             ("bee/b0.png", 200, 130), ("bee/b1.jpg", 64, 64), ("bee/notes.txt", 0, 0),
             ("cat/c0.png", 77, 181), ("cat/c1.jpg", 120, 160)]
    for i, (name, h, w) in enumerate(items):
        p = SRC / name
        if h == 0:
            p.write_text("not an image")
            continue
        im = Image.fromarray(synth_image(200 + i, h, w))
        if name.endswith(".jpg") and i == 7:  # EXIF orientation 6 (rotate 90)
            exif = Image.Exif()
            exif[0x0112] = 6
            im.save(p, quality=92, exif=exif.tobytes())
        elif name.endswith(".jpg"):
            im.save(p, quality=92)
        else:
            im.save(p)
    g = {"builds": []}
    for max_res, q, seed in ((96, 90, 5), (128, 75, 0)):
        out = OUT / f"_tmp_build_{max_res}.essl"
        s = build_container(BuildSpec(SRC, max_res, q, seed), out, workers=2)
        data = out.read_bytes()
        g["builds"].append({"max_resolution": max_res, "quality": q, "seed": seed,
                            "samples": s.sample_count, "total_bytes": s.total_bytes,
                            "bytes": len(data), "sha256": hashlib.sha256(data).hexdigest()})
        out.unlink()
    (OUT / "golden_build.json").write_text(json.dumps(g, indent=1))
    print(g)


if __name__ == "__main__":
    main()
