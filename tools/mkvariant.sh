#!/bin/bash
# Build a variant library = committed csrc/include + a patch (python or sh)
# into _lib<NAME>/, then restore the committed sources.  Needs clean csrc/include.
# Usage: tools/mkvariant.sh NAME PATCH
set -e
cd "$(dirname "$0")/.."
name=$1; patch=$2
git diff --quiet -- paper_2404_00509_b200/csrc include || { echo "csrc/include not clean"; exit 1; }
case "$patch" in *.py) python "$patch";; *) bash "$patch";; esac
python -c "from paper_2404_00509_b200 import build; build.build()"
mkdir -p _lib$name && cp paper_2404_00509_b200/_lib/libessl.so _lib$name/libessl.so
git checkout -q -- paper_2404_00509_b200/csrc include
python -c "from paper_2404_00509_b200 import build; build.build()"
echo "built _lib$name"
