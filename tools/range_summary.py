"""Summarise a pipeline-range ncu report (tools/r2_range.sh) into
profiles/<tag>.json: warp instructions and DRAM bytes per image, issue-slot
and pipe utilisation, warp states.
    python tools/range_summary.py gpurun_out/range_r2a.ncu-rep --images 16384 --out profiles/x.json"""
import argparse
import csv
import io
import json
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--images", type=int, required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    ap.add_argument("--cmd", default="ESSL_PROFILER_RANGE=1 ncu --replay-mode app-range --clock-control none "
                    "--section SpeedOfLight --section SchedulerStats --section WarpStateStats --section "
                    "ComputeWorkloadAnalysis --section MemoryWorkloadAnalysis --section InstructionStats "
                    "python tools/graph_profile.py --streams 8 --batches 64 --replays 1")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    d = dict(zip(rows[0], rows[2]))

    def f(k):
        return float(d[k].replace(",", ""))

    ms = f("gpu__time_duration.sum")
    res = {"cmd": a.cmd, "note": a.note, "duration_ms": ms, "images": a.images,
           "img_per_s_in_range": a.images / (ms / 1e3),
           "warp_instructions_per_image": f("smsp__inst_executed.sum") / a.images,
           "issue_slots_busy_pct": f("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
           "sm_clock_ghz": f("gpc__cycles_elapsed.avg.per_second"),
           "warps_active_per_scheduler": f("smsp__warps_active.avg.per_cycle_active"),
           "eligible_warps_per_scheduler": f("smsp__warps_eligible.avg.per_cycle_active"),
           "dram_tbs": f("dram__bytes.sum.per_second"),
           "pipe_util_pct_active": {p: f(f"sm__pipe_{p}_cycles_active.avg.pct_of_peak_sustained_active")
                                    for p in ("alu", "fma", "fp64", "lsu", "xu", "adu", "cbu", "uniform")
                                    if f"sm__pipe_{p}_cycles_active.avg.pct_of_peak_sustained_active" in d},
           "stall_cycles_per_issue": {}}
    res["dram_bytes_per_image"] = res["dram_tbs"] * 1e12 * ms / 1e3 / a.images
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    for k in d:
        if k.startswith(pre) and k.endswith(suf):
            v = f(k)
            if v > 0.01:
                res["stall_cycles_per_issue"][k[len(pre):-len(suf)]] = round(v, 3)
    json.dump(res, open(a.out, "w"), indent=1)
    print(json.dumps({k: res[k] for k in ("warp_instructions_per_image", "issue_slots_busy_pct",
                                          "dram_bytes_per_image", "img_per_s_in_range")}))


if __name__ == "__main__":
    main()
