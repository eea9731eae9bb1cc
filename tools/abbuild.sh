#!/bin/bash
# Builds an A/B variant of the library: tools/abbuild.sh NAME "-DFLAG=V ..."
# -> abtest/NAME/libgpfilter_b200.so (bench.py / tests pick it via GPF_B200_LIB)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
N=$1; shift
mkdir -p "$ROOT/abtest/$N"
make -s -j8 -C "$ROOT/paper_1505_00077_b200" "$ROOT/abtest/$N/libgpfilter_b200.so" \
  LIB="$ROOT/abtest/$N/libgpfilter_b200.so" OBJDIR="$ROOT/abtest/$N/build" EXTRA_NVFLAGS="$*"
