#!/bin/bash
# K3 pinhole: Horner tile configs vs the direct fast tile (C2: 3 channels, C3: 1 channel)
for cfg in 0 1 2 3 4; do
  FDL_HORNER_CFG=$cfg python bench.py --no-cpu-baseline --no-e2e --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c2 cfg $cfg', round(d['render']['value']), round(d['stages_ms']['k3_render_spectra_ms'],4))"
  FDL_HORNER_CFG=$cfg python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 5 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c3 cfg $cfg', round(d['render']['value']), round(d['stages_ms']['k3_render_spectra_ms'],4))"
done
FDL_RENDER_KERNEL=fast python bench.py --no-cpu-baseline --no-e2e --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c2 direct', round(d['render']['value']), round(d['stages_ms']['k3_render_spectra_ms'],4))"
