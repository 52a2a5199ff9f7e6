# K1 timing (c2, c4) + one ncu capture of k1_fast_kernel on c2
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench_c2.json'));print('c2 construct',d['construct_ms'],'k1',d['k1_ms'],'frac',d['roofline']['frac'],'render',d['render'])"
timeout 600 python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench_c4.json'));print('c4 construct',d['construct_ms'],'k1',d['k1_ms'],'frac',d['roofline']['frac'],'render',d['render'])"
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 1 -c 1 -o gpurun_out/k1_c2 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1.log 2>&1; tail -1 gpurun_out/ncu_k1.log
