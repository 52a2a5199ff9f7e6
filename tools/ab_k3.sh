#!/bin/bash
# K3 pinhole tiles: horner2 (default) / fast (direct) / horner (HB blocks) on C2 (3 ch) and C3 (1 ch)
for rk in 2 fast horner; do
  FDL_RENDER_KERNEL=$rk python bench.py --no-cpu-baseline --no-e2e --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['render'];print('c2 $rk', round(r['value']), 'k3', round(r['roofline']['k3_ms'],4), 'frac', round(r['roofline']['frac'],3))"
  FDL_RENDER_KERNEL=$rk python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 5 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['render'];print('c3 $rk', round(r['value']), 'k3', round(r['roofline']['k3_ms'],4), 'frac', round(r['roofline']['frac'],3))"
done
