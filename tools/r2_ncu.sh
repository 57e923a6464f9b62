#!/bin/bash
# ncu --set full of one kernel of the bench's single-stream launch sequence.
# Usage: bash tools/r2_ncu.sh <kernel regex> <tag> [bench args...]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
K=$1; TAG=$2; shift 2
B="bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --streams 1 $*"
timeout 300 python $B > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$K" -s 5 -c 1 -o gpurun_out/ncu_$TAG python $B > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu $TAG rc=$?"
