"""Build libessl.so in-tree with nvcc for sm_100a.

    python -m paper_2404_00509_b200.build        # or __graft_entry__.build()

Objects are compiled in parallel; the shared library lands in
paper_2404_00509_b200/_lib/libessl.so (git-ignored, travels with gpurun).
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libessl.so"
ARCH = "-gencode=arch=compute_100a,code=sm_100a"

SOURCES = ["decode.cu", "pixels.cu", "api.cu", "host.cpp"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; libessl cannot be built")


CHECKED = os.environ.get("ESSL_CHECKED") == "1"  # bounds-checked variant (_lib/checked/)
if CHECKED:
    OUT_DIR = PKG / "_lib" / "checked"
    LIB = OUT_DIR / "libessl.so"


def _flags(src: str) -> list[str]:
    common = ["-std=c++17", "-O3", "-lineinfo", f"-I{ROOT / 'include'}", f"-I{CSRC}",
              "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math,-fvisibility=hidden"]
    if CHECKED:
        common.append("-DESSL_CHECKED")
    if src.endswith(".cu"):
        # -fmad=false: float64/float32 parity stages must not contract to FMA
        return common + [ARCH, "-fmad=false", "-Xptxas", "-warn-spills"]
    return common


def _digest() -> str:
    h = hashlib.sha256()
    for f in sorted(CSRC.iterdir()):
        if f.suffix in (".cu", ".cuh", ".cpp", ".h"):
            h.update(f.name.encode() + f.read_bytes())
    h.update((ROOT / "include" / "essl.h").read_bytes())
    # flags without the checkout's absolute path: a copied tree (the GPU box)
    # sees the same digest and reuses the shipped library
    flags = " ".join(_flags("x.cu") + _flags("x.cpp")).replace(str(ROOT), "<root>")
    h.update(flags.encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> Path:
    override = os.environ.get("ESSL_LIB")
    if override and not force and not CHECKED:  # an A/B build chosen by the caller: never rebuild over it
        return Path(override)
    OUT_DIR.mkdir(exist_ok=True)
    stamp = OUT_DIR / "libessl.sha256"
    dig = _digest()
    if LIB.exists() and stamp.exists() and stamp.read_text() == dig and not force:
        return LIB
    # one builder at a time (torchrun ranks, parallel test workers): the
    # others wait, then find the stamp current
    import fcntl
    with open(OUT_DIR / ".build.lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        if LIB.exists() and stamp.exists() and stamp.read_text() == dig and not force:
            return LIB
        return _build_locked(dig, stamp, verbose)


def _build_locked(dig: str, stamp: Path, verbose: bool) -> Path:
    nvcc = _nvcc()
    objs = []

    def compile_one(src: str) -> Path:
        obj = OUT_DIR / (src.replace(".", "_") + ".o")
        cmd = [nvcc, *_flags(src), "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr.strip():
            print(r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as pool:
        objs = list(pool.map(compile_one, SOURCES))
    tmp = OUT_DIR / "libessl.so.tmp"
    cmd = [nvcc, "-shared", ARCH, "-o", str(tmp), *map(str, objs), "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stdout}\n{r.stderr}")
    tmp.replace(LIB)
    stamp.write_text(dig)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
