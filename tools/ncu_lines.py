"""Per-source-line executed warp instructions (and stall samples) of an ncu
report's kernel: python tools/ncu_lines.py <rep> [top]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path" or r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            ie = int(d.get("Instructions Executed", "0") or 0)
            ss = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        rows.append((ie, ss, fname, int(r[0]), r[1].strip()[:90]))
tot = sum(r[0] for r in rows) or 1
tots = sum(r[1] for r in rows) or 1
print(f"total warp instructions {tot:,}  stall samples {tots:,}")
for ie, ss, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*ie/tot:5.1f}% {100*ss/tots:5.1f}%  {f}:{ln:<5} {src}")
