"""Command line: ``python -m paper_2404_00509_b200 stream --config loader.json
[--epoch E] [--batches N] [--digest]`` -- the reference's ``cropload stream``
(cli.py:138-211, 281-288) on the GPU loader: the binary batch stream (or
per-batch digests) on stdout, diagnostics on stderr."""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path


def _cmd_stream(args) -> int:
    from .pipeline import Loader, LoaderConfig
    from .stream import digest_stream, write_stream
    doc = json.loads(Path(args.config).read_text())
    cfg = LoaderConfig.from_document(doc)
    cfg.out_dtype = "float32"
    with Loader(cfg) as loader:
        if args.digest:
            for d in digest_stream(loader, args.epoch, args.batches):
                sys.stdout.write(json.dumps(d, separators=(",", ":")) + "\n")
        else:
            out = sys.stdout.buffer
            write_stream(loader, args.epoch, out, args.batches)
            out.flush()
    return 0


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="paper_2404_00509_b200")
    sub = p.add_subparsers(dest="cmd", required=True)
    st = sub.add_parser("stream", help="stream batches as binary frames (bindings surface)")
    st.add_argument("--config", required=True)
    st.add_argument("--epoch", type=int, default=0)
    st.add_argument("--batches", type=int, default=None)
    st.add_argument("--digest", action="store_true")
    st.set_defaults(fn=_cmd_stream)
    args = p.parse_args(argv)
    return args.fn(args)


if __name__ == "__main__":
    sys.exit(main())
