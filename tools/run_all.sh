# round-end style measurement sweep (writes gpurun_out/r01_*)
set -x
python -m pytest tests -m gpu -q -rf > gpurun_out/r01_pytest_gpu.log 2>&1; tail -1 gpurun_out/r01_pytest_gpu.log
python bench.py > gpurun_out/r01_bench_c2.json 2> gpurun_out/r01_bench_c2.err
python bench.py --impl reference > gpurun_out/r01_bench_c2_reference.json 2>&1
python bench.py --config c1 --no-cpu-baseline > gpurun_out/r01_bench_c1.json 2>&1
timeout 900 python bench.py --config c3 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r01_bench_c3.json 2>&1
timeout 900 python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r01_bench_c4.json 2>&1
timeout 900 python bench.py --config c2b --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r01_bench_c2b.json 2>&1
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 > gpurun_out/r01_bench_c5.json 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01_smoke.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 1 -c 1 -o gpurun_out/r01_k1_c2 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:render_pin -s 1 -c 1 -o gpurun_out/r01_k3_c2 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k3.log 2>&1
python bench.py --config c5 --steps 1 --warmup 1 --c5-views 64 > gpurun_out/plain5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:render_tile -s 1 -c 1 -o gpurun_out/r01_k3_c5 -f python bench.py --config c5 --steps 1 --warmup 1 --c5-views 64 > gpurun_out/ncu_k3c5.log 2>&1
