#!/bin/bash
# round-2 baseline: the driver's bench command, plus a longer run for comparison
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nproc; lscpu | grep -E "Model name|Socket|NUMA node\(s\)|^CPU\(s\)"
for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2b_s20_$i.json 2> gpurun_out/r2b_s20_$i.err; echo "s20 rc=$?"
done
timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu > gpurun_out/r2b_s300.json 2> gpurun_out/r2b_s300.err; echo "s300 rc=$?"
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --streams 4 > gpurun_out/r2b_s20_st4.json 2>&1; echo "st4 rc=$?"
for f in gpurun_out/r2b_*.json; do python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print('$f', round(d['value']), round(d['e2e']['value'] or 0), d['ms_per_step'])
"; done
