# Launch lists (cold-cache, serialised) of the headline's two halves, own + cuFFT kernels only.
O=gpurun_out/r02b
mkdir -p $O
M=gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,dram__bytes_read.sum,dram__bytes_write.sum
F='regex:^(?!.*(elementwise|reduce_kernel|distribution|arange|exp_kernel|CatArray|index|fill|copy)).*$'
ncu --metrics $M --clock-control none -k "$F" -c 400 --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c4.log 2>&1
tail -1 $O/ncu_c4.log | head -c 300; echo
ncu --metrics $M --clock-control none -k "$F" -c 400 --csv --log-file $O/launches_c5.csv python bench.py --config c5 --c5-views 256 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c5.log 2>&1
tail -1 $O/ncu_c5.log | head -c 300; echo
