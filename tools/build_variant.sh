#!/bin/bash
# Build an A/B variant of libtnl.so with extra nvcc flags into exp/libtnl_<name>.so, then restore
# the default build.  usage: tools/build_variant.sh <name> "<flags>"
set -e
cd "$(dirname "$0")/.."
mkdir -p exp
TNL_NVCC_EXTRA="$2" python -m paper_2602_01613_b200.build --force >/dev/null
cp paper_2602_01613_b200/libtnl.so "exp/libtnl_$1.so"
python -m paper_2602_01613_b200.build --force >/dev/null
