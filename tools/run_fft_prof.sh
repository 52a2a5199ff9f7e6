ncu --set full --import-source on --clock-control none -k regex:"fwd_cols" -c 1 -o gpurun_out/fft_full3 python bench.py --config c2 --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > gpurun_out/ncu_fft_full.log 2>&1
tail -1 gpurun_out/ncu_fft_full.log
