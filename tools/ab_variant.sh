#!/bin/bash
# Build the working tree's library into _libB/ (variant B) and the committed
# sources' (HEAD) into _libA/ (variant A); paper_2404_00509_b200/_lib is left
# holding the working tree's build.  Compare with
#   python tools/ab.py --a _libA/libessl.so --b _libB/libessl.so
# (ESSL_LIB makes build() load that file and never rebuild over it).
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2404_00509_b200 import build; build.build()"
mkdir -p _libB _libA && cp paper_2404_00509_b200/_lib/libessl.so _libB/libessl.so
git stash -q
python -c "from paper_2404_00509_b200 import build; build.build()"
cp paper_2404_00509_b200/_lib/libessl.so _libA/libessl.so
git stash pop -q
python -c "from paper_2404_00509_b200 import build; build.build()"
echo "A: _libA/libessl.so (HEAD), B: _libB/libessl.so (working tree)"
