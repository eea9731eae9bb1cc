#!/bin/bash
# GPU A/B session: parity tests on the default build, then the bench A/B of
# the variants given as arguments (abtest/NAME or "base"), AB_ROUNDS rounds.
# usage: tools/gpu_ab.sh OUTPREFIX "pytest args" VARIANT...
OUT=$1; shift; PT=$1; shift
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${OUT}_smi.txt
if [ -n "$PT" ]; then
  timeout 1200 python -m pytest $PT -x -q > gpurun_out/${OUT}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${OUT}_pytest.log
  tail -3 gpurun_out/${OUT}_pytest.log
fi
bash tools/ab_bench.sh "$OUT" "$@" 2>&1 | tee gpurun_out/${OUT}_ab.txt
