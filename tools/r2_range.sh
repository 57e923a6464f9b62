#!/bin/bash
# Pipeline-range ncu: the 8-stream loader captured in a CUDA graph, measured
# as one app range (issue slots, warp states, DRAM of the concurrent mix).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${1:-range}
CMD="python tools/graph_profile.py --streams 8 --batches 64 --replays 1"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ESSL_PROFILER_RANGE=1 timeout 900 ncu --replay-mode app-range --clock-control none --section SpeedOfLight --section SchedulerStats --section WarpStateStats --section ComputeWorkloadAnalysis --section MemoryWorkloadAnalysis --section InstructionStats -o gpurun_out/$TAG $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "range rc=$?"
cat gpurun_out/${TAG}_plain.log | tail -2
