#!/bin/bash
# Same-box A/B of library variants on the bench (C3 five-sigma_s step):
#   tools/ab_bench.sh OUTPREFIX base abtest/NAME1 abtest/NAME2 ...  (alternating, 2 rounds)
OUT=$1; shift
for round in ${AB_ROUNDS:-1 2}; do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=""; else lib="$v/libgpfilter_b200.so"; fi
    tag=$(basename "$v")
    GPF_B200_LIB=$lib python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline --no-mse \
      > "gpurun_out/${OUT}_${tag}_${round}.json" 2> "gpurun_out/${OUT}_${tag}_${round}.err"
    python - "gpurun_out/${OUT}_${tag}_${round}.json" "$tag" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], d["value"], "stage", d["stage_ms_per_frame"], "clk", d["clocks"]["sm_mhz"], "W", d["clocks"].get("power_w"))
PY
  done
done
