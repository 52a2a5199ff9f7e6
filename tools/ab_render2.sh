#!/bin/bash
# A/B of the K3 render tiles: legacy (round-1) vs fast; C2 (pinhole, 3 ch), C3 (pinhole, 1 ch), C5 (disk aperture)
set -u
mkdir -p gpurun_out
for impl in legacy fast; do
  FDL_RENDER_KERNEL=$impl python bench.py --no-cpu-baseline --no-e2e --steps 10 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c2', '$impl', d['render'], d['stages_ms'])"
  FDL_RENDER_KERNEL=$impl python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 5 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c3', '$impl', d['render'], d['stages_ms'])"
  FDL_RENDER_KERNEL=$impl python bench.py --config c5 --steps 3 --warmup 2 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c5', '$impl', d['value'], d.get('render_flops_tf'), d.get('stages_ms'))"
done
