#!/bin/bash
# per-kernel durations of one fp64-mode call (ncu launch list), C5 by default
c=${1:-5}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/fp64_one.py $c 1 2>/dev/null | python -c "
import csv,sys
rows=[l for l in sys.stdin if l.startswith('\"')]
for r in csv.DictReader(rows):
    print(r['Kernel Name'].split('(')[0][-24:], r['Metric Value'])
"
