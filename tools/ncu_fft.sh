O=gpurun_out/r02p
mkdir -p $O
ncu --set full --import-source on --clock-control none -k regex:"fwd_rows|fwd_cols|inv_cols|inv_rows" -s 8 -c 4 -o $O/fft python tools/bench_fft.py 2048 48 48 > $O/ncu.log 2>&1
tail -2 $O/ncu.log
