# source-level ncu capture of the C2 FFT column/row kernels (forward cols, inverse rows)
O=gpurun_out/fftsrc
mkdir -p $O
python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"fwd_cols|inv_rows|fwd_rows|inv_cols" -c 4 -o $O/fft python bench.py --config c2 --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > $O/ncu.log 2>&1
tail -2 $O/ncu.log
