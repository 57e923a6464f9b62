#!/bin/bash
# Interleaved bench A/B over option sets: bash tools/r2_ab.sh "<args A>" "<args B>" ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
STEPS=${STEPS:-300}
REPS=${REPS:-2}
for rep in $(seq $REPS); do
  i=0
  for a in "$@"; do
    timeout 300 python bench.py --steps $STEPS --warmup 5 --no-cpu $a > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
    python -c "
import json
for l in open('gpurun_out/ab_$i.json'):
    if l.startswith('{'):
        d=json.loads(l); print('rep $rep [$a]', round(d['value']), 'e2e', round(d['e2e']['value'] or 0), {k: round(v,4) for k,v in d['roofline']['kernel_ms'].items()})
" || tail -5 gpurun_out/ab_$i.err
    i=$((i+1))
  done
done
