python -m pytest tests -m gpu -q -x -s 2>&1 | grep -E "rel L2|passed|failed|Error" | head -30
python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1; tail -c 1500 gpurun_out/bench_c2.json; echo
timeout 600 python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2>&1; tail -c 1200 gpurun_out/bench_c4.json; echo
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 1 -c 1 -o gpurun_out/k1_c2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1.log 2>&1; tail -3 gpurun_out/ncu_k1.log
