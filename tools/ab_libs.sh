#!/bin/bash
# Build an honest A/B pair for the GPU box: build/base = the committed sources
# (HEAD), build/var = the working tree.  (tools/variant.py rebuilds the
# in-tree library from the working tree first, so a variant built with it is
# NOT compared against HEAD unless the base library is saved like this.)
set -e
cd "$(dirname "$0")/.."
rm -rf build/base build/var
mkdir -p build/base build/var
git stash push -q -- paper_1912_07645_b200/csrc
python -m paper_1912_07645_b200.build > /dev/null
cp paper_1912_07645_b200/_lib/libfvb200.so build/base/
git stash pop -q
python -m paper_1912_07645_b200.build > /dev/null
cp paper_1912_07645_b200/_lib/libfvb200.so build/var/
cmp -s build/base/libfvb200.so build/var/libfvb200.so && echo "WARNING: base and var identical" || echo "base and var differ"
