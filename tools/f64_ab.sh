#!/bin/bash
# fp64 mode A/B on one box: device time of C5 and C2 for the default build and
# the variants built by tools/abbuild.sh (abtest/NAME). usage: tools/f64_ab.sh NAME...
for i in 1 2; do
  for c in 5 2; do
    python tools/fp64_one.py $c 3 | tail -1 | sed 's/^/base /'
    for v in "$@"; do
      GPF_B200_LIB=abtest/$v/libgpfilter_b200.so python tools/fp64_one.py $c 3 | tail -1 | sed "s/^/$v /"
    done
  done
done
