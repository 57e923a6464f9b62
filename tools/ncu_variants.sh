#!/bin/bash
# One ncu over several libessl builds: k_entropy's 6th launch of each (source
# counters: per-SASS executed instructions).  Usage: bash tools/ncu_variants.sh TAG lib1 lib2 ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
tag=$1; shift
mkdir -p gpurun_out
cat > /tmp/nv_run.sh <<EOS
for lib in $@; do
  ESSL_LIB=\$PWD/\$lib timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --streams 1 > /dev/null 2>&1
done
EOS
timeout 1200 ncu --kernel-id "::regex:k_entropy:6" --section SourceCounters --section InstructionStats \
  --section LaunchStats --section SpeedOfLight --section Occupancy --import-source on --clock-control none \
  -o gpurun_out/${tag}_nv -f bash /tmp/nv_run.sh > gpurun_out/${tag}_nv.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${tag}_nv.log
