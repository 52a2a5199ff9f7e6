# A/B of the affine aperture tile's views per thread / CTAs per SM (rebuilds the library on the GPU box)
for cfg in "8 2" "6 2" "4 3" "4 4"; do
  set -- $cfg
  FDL_NVCC_EXTRA="-DFDL_AP_VB3=$1 -DFDL_AP_MINB=$2" python -c "
from paper_1901_06919_b200 import build_native as b; b.build(force=True, verbose=False)" > /dev/null 2>&1
  python bench.py --config c5 --c5-views 512 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('VB $1 minb $2:', d['roofline']['kernel_ms_per_launch'], d['stages_ms'])"
done
