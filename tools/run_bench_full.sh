# full default bench (driver contract) + reference arm + NVTX-filtered launch list
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 3000 gpurun_out/bench_default.json; echo
python bench.py --impl reference > gpurun_out/bench_reference.json 2>&1; tail -c 1500 gpurun_out/bench_reference.json; echo
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_timed_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log
