#!/bin/bash
# Round-2 evidence pass: bench lines (driver command + 300 steps), the launch
# list, one ncu --set full per kernel (single-stream bench, 256 images per
# launch) and the pipeline-range ncu.  Each ncu only after its command ran clean.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench20.json 2> gpurun_out/${TAG}_bench20.err; echo "bench20 rc=$?"
timeout 600 python bench.py --steps 300 --warmup 5 --no-cpu > gpurun_out/${TAG}_bench300.json 2> gpurun_out/${TAG}_bench300.err; echo "bench300 rc=$?"
B="bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --streams 1 --group 1"
timeout 300 python $B > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python $B > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "launch list rc=$?"
for k in ${KERNELS:-k_entropy k_prep k_idct k_resize k_mask}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^$k" -s 5 -c 1 -o gpurun_out/${TAG}_ncu_$k python $B > gpurun_out/${TAG}_ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
bash tools/r2_range.sh ${TAG}_range
