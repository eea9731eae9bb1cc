#!/bin/bash
# Run-to-run spread of the default bench on one box (wall time of each run) and the C4 workload.
T=${1:-runs}
for i in 1 2 3; do
  s=$(date +%s)
  python bench.py > gpurun_out/${T}_bench_run$i.json 2> gpurun_out/${T}_bench_run$i.err
  rc=$?; e=$(date +%s); echo "run $i rc $rc wall $((e - s)) s"
done
python bench.py --workload c4 > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err; echo "c4 rc $?"
python - "$T" <<'PY'
import json, sys
T = sys.argv[1]
for f in ["bench_run1", "bench_run2", "bench_run3", "bench_c4"]:
    d = json.loads(open(f"gpurun_out/{T}_{f}.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f, d["value"], r.get("step", r)["frac"], d["e2e"]["value"], d["clocks"])
PY
