# A/B of the TMA aperture tile (1 or 2 view groups per CTA) against the round-1 tile on C5.
O=gpurun_out/r02c
mkdir -p $O
python -m pytest tests -m gpu -q -x -k "apert or c5 or render or fullsize" > $O/pytest_render.log 2>&1; tail -3 $O/pytest_render.log
for g in 1 2; do
  FDL_AP_GROUPS=$g python bench.py --config c5 --c5-views 1024 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_c5_g$g.json 2> $O/bench_c5_g$g.err
  python - <<PY
import json
d=json.loads(open("$O/bench_c5_g$g.json").read().strip().splitlines()[-1])
print("groups $g", d["value"], d.get("stages_ms"), d.get("roofline",{}).get("frac"), d.get("roofline",{}).get("kernel_ms_per_launch"))
PY
done
FDL_RENDER_KERNEL=legacy python bench.py --config c5 --c5-views 1024 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_c5_legacy.json 2> $O/bench_c5_legacy.err
python - <<PY
import json
d=json.loads(open("$O/bench_c5_legacy.json").read().strip().splitlines()[-1])
print("legacy", d["value"], d.get("stages_ms"), d.get("roofline",{}).get("frac"), d.get("roofline",{}).get("kernel_ms_per_launch"))
PY
