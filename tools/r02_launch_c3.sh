O=gpurun_out/r02n
mkdir -p $O
M=gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,dram__bytes_read.sum,dram__bytes_write.sum
for c in c3 c2; do
ncu --metrics $M --clock-control none -k regex:"k1_|count_status|screen|symmetrize|fwd_|inv_|render_|sumsq|lambda" -c 60 --csv --log-file $O/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_$c.log 2>&1
done
