"""Per-result hot-loop summary of an ncu report with SourceCounters (SASS
view): total warp instructions and the regions (contiguous hot SASS) that
execute them, for each profiled kernel instance.
    python tools/sass_hot.py report.ncu-rep [--min 0.01] [--dump N]"""
from __future__ import annotations

import argparse
import csv
import io
import subprocess


def blocks(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    cur = []
    for line in out.splitlines():
        if line.startswith('"Kernel Name"') and cur:
            yield cur
            cur = []
        cur.append(line)
    if cur:
        yield cur


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--min", type=float, default=0.01)
    ap.add_argument("--dump", type=int, default=-1, help="print the SASS of hot region N of each result")
    a = ap.parse_args()
    for bi, lines in enumerate(blocks(a.rep)):
        rows = list(csv.reader(io.StringIO("\n".join(lines))))
        name, hdr, data = rows[0][1], rows[1], rows[2:]
        ie = hdr.index("Instructions Executed")
        cnt = [int(r[ie] or 0) for r in data]
        tot = sum(cnt)
        print(f"[{bi}] {name}: {tot:,} warp instructions")
        hot = [i for i, c in enumerate(cnt) if c > tot * 0.002]
        runs = []
        for i in hot:
            if runs and i - runs[-1][1] <= 3:
                runs[-1][1] = i
            else:
                runs.append([i, i])
        for ri, (s, e) in enumerate(runs):
            c = sum(cnt[s:e + 1])
            if c < tot * a.min:
                continue
            iters = max(cnt[s:e + 1])
            print(f"   region {ri}: SASS {s}-{e} ({e - s + 1} instr) {c / tot * 100:5.1f}% of instr, "
                  f"max count {iters:,} -> {c / max(iters, 1):.1f} instr/iteration")
            if ri == a.dump:
                for i in range(s, e + 1):
                    print(f"      {cnt[i]:>10} {data[i][1]}")


if __name__ == "__main__":
    main()
