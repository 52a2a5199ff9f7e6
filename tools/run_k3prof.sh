#!/bin/bash
# one ncu --set full capture of the K3 render tile for C2 (pinhole Horner) and C5 (disk aperture)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:render_horner -s 1 -c 1 -o gpurun_out/k3h_c2 -f \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k3h_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:render_ap_fast -s 1 -c 1 -o gpurun_out/k3f_c5 -f \
  python bench.py --config c5 --c5-views 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k3f_c5.log 2>&1
