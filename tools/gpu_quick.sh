#!/bin/bash
# GPU tests (quiet) + decode sweep summary.  Usage: bash tools/gpu_quick.sh [sweep-args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 400 python tools/decode_bench.py "$@" > gpurun_out/dbench.log 2>&1; echo "dbench rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/dbench.log"):
    if l.startswith("{"):
        d = json.loads(l)
        ph = d["phase_kcycles_median"]
        print(d["mode"], d["seq_bits"], d["warm_bits"], "decode_ms %.3f" % d["decode_ms"],
              {k: ph[k] for k in ("prep", "count", "continuation", "resolve", "write_fixup")},
              "cont", d["cont_bits_max_median"], "units", d.get("units_phase1_mean"), "guess", d.get("reguess_phase1_mean"), "lane_max_units", d.get("units_phase1_lane_max_median"), "fallback", d.get("fallback_images"))
PY
