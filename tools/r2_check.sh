#!/bin/bash
# GPU tests (quiet) + short benches.  Usage: bash tools/r2_check.sh [pytest -k expr]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
K=${1:-}
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -x -q -m gpu -k "$K" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
else
  timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
fi
tail -25 gpurun_out/pytest_gpu.log
for s in 20 300; do
  timeout 300 python bench.py --steps $s --warmup 5 --no-cpu > gpurun_out/b_s$s.json 2> gpurun_out/b_s$s.err; echo "bench s$s rc=$?"
  tail -3 gpurun_out/b_s$s.err
  python -c "
import json
for l in open('gpurun_out/b_s$s.json'):
    if l.startswith('{'):
        d=json.loads(l); print('s$s value', round(d['value']), 'e2e', round(d['e2e']['value'] or 0), 'ms/step', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['roofline']['kernel_ms'].items()})
"
done
