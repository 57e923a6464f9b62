"""Summarise ncu reports (--set full captures) into small JSON files for
profiles/: duration, DRAM bytes, throughputs, issue activity, occupancy
and the warp-stall breakdown of the captured kernel.

    python tools/ncu_summary.py gpurun_out/ncu_k_entropy.ncu-rep ... --out-dir profiles --tag r1
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

RAW = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__inst_issued.avg.pct_of_peak_sustained_active": "inst_issued_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_static": "smem_static",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic",
    "sm__cycles_active.avg": "sm_active_cycles",
    "gpc__cycles_elapsed.max": "elapsed_cycles",
}


def summarize(rep: Path) -> dict:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    scale = {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
             "second": 1e9, "s": 1e9, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
             "Kbyte/block": 1e3, "byte/block": 1}
    res = {"report": rep.name, "kernel": d.get("Kernel Name", ""),
           "units": "time ns, bytes B, smem B"}
    for k, name in RAW.items():
        if k in d:
            try:
                res[name] = float(d[k].replace(",", "")) * scale.get(u.get(k, ""), 1)
            except ValueError:
                res[name] = d[k]
    stalls = {}
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    for k, v in d.items():
        if k.startswith(pre) and k.endswith(suf) and "not_issued" not in k:
            try:
                stalls[k[len(pre):-len(suf)]] = float(v)
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    res["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]}
    if "dram_read_bytes" in res and "dram_write_bytes" in res:
        res["dram_bytes"] = res["dram_read_bytes"] + res["dram_write_bytes"]
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+")
    ap.add_argument("--out-dir", default="profiles")
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    for r in args.reports:
        s = summarize(Path(r))
        s["note"] = args.note
        name = Path(r).stem.replace("ncu_", "")
        p = Path(args.out_dir) / f"{args.tag}_ncu_{name}.json"
        p.write_text(json.dumps(s, indent=1))
        print(p, {k: s.get(k) for k in ("duration_ns", "dram_bytes", "issue_active_pct")})


if __name__ == "__main__":
    main()
