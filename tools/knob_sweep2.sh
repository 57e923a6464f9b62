#!/bin/bash
# bench.py device throughput over (seq_bits, warm_bits).  Usage: bash tools/knob_sweep2.sh "seqs" "warms"
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for s in $1; do for w in $2; do
  timeout 200 python bench.py --no-cpu --no-e2e --seq-bits $s --warm-bits $w > gpurun_out/ks.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ks.json')); print($s, $w, round(d['value']), {k: round(v,3) for k,v in d['roofline']['kernel_ms'].items()})"
done; done
