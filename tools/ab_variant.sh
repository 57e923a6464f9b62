#!/bin/bash
# Build the working tree's library into _libB/ (variant B) and restore the
# committed sources' build in paper_2404_00509_b200/_lib (variant A).
# Usage: make the B edit, run tools/ab_variant.sh, then revert the edit is done here (git stash).
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2404_00509_b200 import build; build.build()"
mkdir -p _libB && cp paper_2404_00509_b200/_lib/libessl.so _libB/libessl.so
git stash -q
python -c "from paper_2404_00509_b200 import build; build.build()"
git stash pop -q
echo "A: paper_2404_00509_b200/_lib/libessl.so (HEAD), B: _libB/libessl.so (working tree)"
