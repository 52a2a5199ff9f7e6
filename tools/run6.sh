set -x
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -3 gpurun_out/bench_c2.err
cat gpurun_out/bench_c2.json
python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2>&1; cat gpurun_out/bench_c1.json | tail -2
timeout 600 python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2>&1; tail -2 gpurun_out/bench_c4.json
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu.log 2>&1; tail -3 gpurun_out/ncu.log
