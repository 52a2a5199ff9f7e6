#!/bin/bash
# C5 (disk aperture renders): aperture Horner tile (opt-in) vs the round-1 tile (default) vs the fast direct tile
for rk in aph legacy fast; do
  FDL_RENDER_KERNEL=$rk python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c5 $rk', round(d['value']), 'k3', round(d['stages_ms']['k3_render_spectra_ms'],3), 'frac', round(d['roofline']['frac'],3))"
done
