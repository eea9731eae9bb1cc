#!/bin/bash
# Same-box A/B of bench environment settings: tools/ab_env.sh OUT "VAR=a" "VAR=b" ... (3 rounds)
OUT=$1; shift
for round in ${AB_ROUNDS:-1 2 3}; do
  for v in "$@"; do
    tag=$(echo "$v" | tr '= ' '__')
    env $v python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline --no-mse \
      > "gpurun_out/${OUT}_${tag}_${round}.json" 2> "gpurun_out/${OUT}_${tag}_${round}.err"
    python - "gpurun_out/${OUT}_${tag}_${round}.json" "$tag" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[2], d["value"], "clk", d["clocks"]["sm_mhz"])
PY
  done
done
