"""Generate the 3-Aug / 3-Aug+ golden fixtures from the
REFERENCE implementation.

Run in the build container (the reference is importable there, it is not on
the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_aug.py

Inputs are stored verbatim (aug_arrays.npz) so the fixtures do not depend on
the reference being importable; expected outputs are SHA-256 digests of the
reference's own results (cropload/imgops.py:75-227, pipeline.py:78-101,
Loader pipeline.py:219-235).  Blur weights come from numpy's exp, whose
result can depend on the host's SIMD level, so every blur record stores the
exact weights (float.hex) next to the digest; tests compare weights first.

Outputs: golden_aug.json, aug_arrays.npz (both under tests/golden/).
"""

from __future__ import annotations

import hashlib
import json
import math
import sys
from pathlib import Path

import numpy as np

from cropload import imgops, rng as R
from cropload.pipeline import Loader, LoaderConfig, apply_aug, sample_rrc
from cropload.schedule import AugLevel
from cropload.synth import synth_image

OUT = Path(__file__).resolve().parent


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def blur_weights(sigma: float):
    """The weights gaussian_blur builds (imgops.py:157-163)."""
    radius = max(1, math.ceil(3.0 * sigma))
    xs = np.arange(-radius, radius + 1, dtype=np.float64)
    wts = np.exp(-(xs * xs) / (2.0 * sigma * sigma))
    wts /= wts.sum()
    return radius, [float(w).hex() for w in wts]


def draws(rng: R.SampleRng, level: AugLevel) -> dict:
    """Replay apply_aug's draws (pipeline.py:85-101) on a copy of the stream."""
    d = {"flip": int(rng.random() < 0.5), "op": -1, "sigma": None, "jitter": None}
    if level is not AugLevel.SIMPLE:
        d["op"] = rng.randint(3)
        if d["op"] == 2:
            d["sigma"] = float(rng.uniform(*imgops.BLUR_SIGMA_RANGE)).hex()
    if level is AugLevel.THREE_AUG_PLUS:
        s = imgops.JITTER_STRENGTH
        d["jitter"] = [float(rng.uniform(1.0 - s, 1.0 + s)).hex() for _ in range(3)]
    return d


def loader_golden(path: Path, cfg_kw: dict, epochs):
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
                    d = draws(rng, loader.aug_level)
                    if d["sigma"] is not None:
                        d["radius"], d["weights"] = blur_weights(float.fromhex(d["sigma"]))
                    recs.append({
                        "epoch": e, "index": idx, "label": int(b.labels[s]),
                        "rect": [r.x, r.y, r.w, r.h], **d,
                        "pixels": sha(b.pixels[s]),
                        "uint8": sha(b.uint8[s]) if b.uint8 is not None else None,
                        "mask": b.mask[s].tolist() if b.mask is not None else None,
                    })
    return recs


def main():
    g: dict = {"generator": "tests/golden/make_golden_aug.py (reference cropload 0.1.0)"}
    arrays: dict = {}
    rr = np.random.default_rng(23)
    srcs = {
        "rand_37x61": rr.integers(0, 256, (37, 61, 3), dtype=np.uint8),
        "rand_16x16": rr.integers(0, 256, (16, 16, 3), dtype=np.uint8),
        "synth_96": synth_image(41, 96, 96),
        "synth_50x70": synth_image(43, 50, 70),
        "gray_ramp": np.repeat(np.arange(0, 256, dtype=np.uint8).reshape(16, 16)[:, :, None],
                               3, 2),
    }
    arrays.update({f"src_{k}": v for k, v in srcs.items()})

    # ---- point ops (imgops.py:75-106, 166-218) ---------------------------------
    ops = {}
    for k, img in srcs.items():
        e = {"grayscale": sha(imgops.grayscale(img)), "solarize": sha(imgops.solarize(img)),
             "luma_mean": float(imgops._luma_mean(img)).hex(), "blur": [], "jitter": []}
        for sigma in (0.1, 0.3333, 0.5, 0.77, 1.0, 1.5, 1.9999):
            radius, wts = blur_weights(sigma)
            e["blur"].append({"sigma": float(sigma).hex(), "radius": radius, "weights": wts,
                              "sha": sha(imgops.gaussian_blur(img, sigma))})
        for f in (0.7, 0.95, 1.0, 1.2345, 1.3):
            e["jitter"].append({"factor": float(f).hex(),
                                "brightness": sha(imgops.adjust_brightness(img, f)),
                                "contrast": sha(imgops.adjust_contrast(img, f)),
                                "saturation": sha(imgops.adjust_saturation(img, f))})
        ops[k] = e
    g["ops"] = ops

    # ---- apply_aug over the rng (pipeline.py:78-101) ----------------------------
    img = srcs["synth_96"]
    g["apply_aug"] = []
    for level in (AugLevel.SIMPLE, AugLevel.THREE_AUG, AugLevel.THREE_AUG_PLUS):
        for i in range(24):
            d = draws(R.SampleRng(1, 2, i), level)
            if d["sigma"] is not None:
                d["radius"], d["weights"] = blur_weights(float.fromhex(d["sigma"]))
            out = apply_aug(R.SampleRng(1, 2, i), img, level)
            g["apply_aug"].append({"level": level.value, "seed": 1, "epoch": 2, "index": i,
                                   **d, "sha": sha(out)})

    # ---- Loader end-to-end ------------------------------------------------------
    g["loader"] = {
        "cfg1_3aug_224": {"data": "cfg1_small.essl",
                          "cfg": dict(batch_size=8, seed=5, res=224, aug="3aug"),
                          "epochs": [0]},
        "cfg1_3augp_224_mask": {"data": "cfg1_small.essl",
                                "cfg": dict(batch_size=8, seed=6, res=224, aug="3aug+",
                                            mask_ratio=0.75, patch=16, keep_uint8=True),
                                "epochs": [1]},
        "mixed_3augp_96_u8": {"data": "mixed_small.essl",
                              "cfg": dict(batch_size=5, seed=77, res=96, aug="3aug+",
                                          keep_uint8=True), "epochs": [4]},
        "cfg4_3aug_160": {"data": "cfg4_small.essl",
                          "cfg": dict(batch_size=4, seed=9, res=160, aug="3aug",
                                      scale=(0.2, 1.0)), "epochs": [0, 1]},
    }
    for key, spec in g["loader"].items():
        spec["samples"] = loader_golden(OUT / spec["data"], spec["cfg"], spec["epochs"])
        spec["cfg"] = {k: (list(v) if isinstance(v, tuple) else v) for k, v in spec["cfg"].items()}
        print(key, len(spec["samples"]), file=sys.stderr)

    (OUT / "golden_aug.json").write_text(json.dumps(g, indent=1))
    np.savez_compressed(OUT / "aug_arrays.npz", **arrays)
    print("wrote", OUT, file=sys.stderr)


if __name__ == "__main__":
    main()
