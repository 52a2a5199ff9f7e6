O=gpurun_out/r02t
mkdir -p $O
ncu --set full --import-source on --clock-control none -k regex:"render_ap_aff" -c 1 -o $O/c5_k3 python bench.py --config c5 --c5-views 256 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_c5.log 2>&1
tail -1 $O/ncu_c5.log | head -c 100; echo
