#!/bin/bash
# Every BASELINE config as a bench line (gpurun_out/bench_<cfg>.json), plus
# the reference (CPU) arm on the default workload.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
run() { name=$1; shift; timeout ${T:-900} python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name rc=$?"; tail -c 600 gpurun_out/bench_$name.json; echo; }
run cfg2 ${CFG2_ARGS}
run ref --impl reference --steps 5 --warmup 3
run cfg1 --workload cfg1 --no-cpu
run cfg3 --workload cfg3 --steps 200 --no-cpu
run cfg4 --workload cfg4 --steps 40 --warmup 5 --pool 4096 --no-cpu
run cfg5 --workload cfg5 --epoch --no-cpu
run cfg2_3aug --aug 3aug --no-cpu
