# source-level ncu capture of the C5 aperture render tile
O=gpurun_out/k3c5
mkdir -p $O
python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"render_tile|render_factors" -c 2 -o $O/k3 python bench.py --config c5 --no-cpu-baseline --no-e2e --steps 1 --warmup 1 --c5-views 64 > $O/ncu.log 2>&1
tail -1 $O/ncu.log
