#!/bin/bash
# K1 stage times on C1/C2/C3 (+ C2b) from bench.py stage timings
for cfg in c2 c3 c2b; do
  python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 5 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$cfg', 'k1_ms', round(d['stages_ms']['k1_ms'],4), 'frac', round(d['roofline']['frac'],3), 'construct_ms', round(d['construct_ms'],3))"
done
