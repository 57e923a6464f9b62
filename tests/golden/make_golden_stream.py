"""Golden batch stream (f4 wire format): the reference's ``cropload stream``
on the committed cfg1_small container, binary and --digest.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_stream.py
"""
import hashlib
import json
import subprocess
import sys
import tempfile
from pathlib import Path

OUT = Path(__file__).resolve().parent
CFG = {"data": "cfg1_small.essl", "batch_size": 16, "workers": 2, "seed": 9, "res": 96,
       "scale": [0.2, 1.0], "ratio": [0.75, 4 / 3], "aug": "simple", "mask_ratio": 0.75, "patch": 16}


def main():
    d = Path(tempfile.mkdtemp())
    cfg = dict(CFG, data=str(OUT / CFG["data"]))
    (d / "cfg.json").write_text(json.dumps(cfg))
    g = {"config": CFG, "runs": []}
    for epoch, nb in ((1, 3), (0, 2)):
        base = [sys.executable, "-m", "cropload", "stream", "--config", str(d / "cfg.json"),
                "--epoch", str(epoch), "--batches", str(nb)]
        raw = subprocess.run(base, capture_output=True, check=True).stdout
        dig = subprocess.run(base + ["--digest"], capture_output=True, check=True, text=True).stdout
        # header + per-batch metas verbatim (the framing), the whole stream as a digest
        g["runs"].append({"epoch": epoch, "batches": nb, "bytes": len(raw),
                          "sha256": hashlib.sha256(raw).hexdigest(),
                          "head": raw[:256].hex(),
                          "digests": [json.loads(x) for x in dig.strip().splitlines()]})
    (OUT / "golden_stream.json").write_text(json.dumps(g, indent=1))
    print("ok", [r["bytes"] for r in g["runs"]])


if __name__ == "__main__":
    main()
