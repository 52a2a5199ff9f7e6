# One full ncu capture each of the C4 K0 passes and of the C5 aperture tile.
O=gpurun_out/r02d
mkdir -p $O
ncu --set full --import-source on --clock-control none -k regex:"fwd_rows_kernel|fwd_cols_kernel" -c 2 -o $O/c4_k0 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_c4.log 2>&1
tail -1 $O/ncu_c4.log | head -c 200; echo
ncu --set full --import-source on --clock-control none -k regex:"render_ap_tma" -c 1 -o $O/c5_k3 python bench.py --config c5 --c5-views 256 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_c5.log 2>&1
tail -1 $O/ncu_c5.log | head -c 200; echo
ls -la $O
