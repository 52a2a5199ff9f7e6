python -m pytest tests/test_gpu_fft.py -q -rf > gpurun_out/pytest_fft.log 2>&1; tail -1 gpurun_out/pytest_fft.log
for c in c2 c4; do
python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/fb_$c.json 2>gpurun_out/fb_$c.err
python -c "import json;d=json.load(open('gpurun_out/fb_$c.json'));print('$c', d['construct_ms'], d['stages_ms'], d['render'])"
done
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"fwd_|inv_" --csv --log-file gpurun_out/fft_launches.csv python bench.py --config c2 --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > gpurun_out/ncu_fft.log 2>&1
python tools/launch_table.py gpurun_out/fft_launches.csv
