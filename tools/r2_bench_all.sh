#!/bin/bash
# Round-2 bench line per BASELINE config (300-step device-timed regions unless
# noted; the driver's own command is 20 steps), gpurun_out/r2_bench_<cfg>.json
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
run() { name=$1; shift; timeout ${T:-900} python bench.py "$@" > gpurun_out/r2_bench_$name.json 2> gpurun_out/r2_bench_$name.err; echo "$name rc=$?"; python -c "
import json,sys
d=json.loads(open('gpurun_out/r2_bench_$name.json').read().strip().splitlines()[-1]); print('$name', round(d['value']), round((d.get('e2e') or {}).get('value') or 0))" ; }
run cfg1 --workload cfg1 --no-cpu --steps 300
run cfg3 --workload cfg3 --steps 300 --no-cpu
run cfg4 --workload cfg4 --steps 40 --warmup 5 --pool 4096 --no-cpu
run cfg5 --workload cfg5 --epoch --no-cpu
run cfg2_3aug --aug 3aug --no-cpu --steps 300
run cfg2_3augplus --aug 3aug+ --no-cpu --steps 300
run cfg2_restart4 --restart 4 --no-cpu --steps 300
