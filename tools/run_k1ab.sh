# K1 A/B: parity tests, C2/C4 K1 timing, ncu of the C2 K1 kernel
O=gpurun_out/k1ab
mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_helpers.py -q -rf -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for c in c2 c4; do
  python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "import json; j=json.load(open('$O/bench_$c.json')); print('$c', 'k1_ms %.3f frac %.3f construct %.3f' % (j['k1_ms'], j['roofline']['frac'], j['construct_ms']))"
done
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 1 -c 1 -o $O/k1_c2 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1; tail -1 $O/ncu.log
