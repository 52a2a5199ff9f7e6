O=gpurun_out/r02p
mkdir -p $O
ncu --set full --import-source on --clock-control none -k regex:"inv_cols|inv_rows" -s 2 -c 2 -o $O/fft_inv python tools/bench_fft.py 2048 48 48 > $O/ncu_inv.log 2>&1
tail -2 $O/ncu_inv.log
