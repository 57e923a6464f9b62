#!/bin/bash
# One gpurun session of evidence: GPU tests, bench line, launch list and one
# ncu --set full capture per kernel (each after its command exited 0 alone).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
B="bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --streams 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python $B > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
for k in ${KERNELS:-k_entropy k_prep k_idct k_resize k_mask}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^$k" -s 5 -c 1 -o gpurun_out/ncu_$k python $B > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
