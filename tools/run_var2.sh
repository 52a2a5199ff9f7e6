# A/B prebuilt variants/*.so: parity (parity file) + C2/C4 K1 time
for v in variants/*.so; do
  cp $v paper_1901_06919_b200/_lib/libfdl_b200.so
  python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
  for c in ${CONFIGS:-c2 c4}; do
    python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/v.json 2>gpurun_out/v.err
    python -c "import json;d=json.load(open('gpurun_out/v.json'));print('$v $c', 'k1 %.3f frac %.3f construct %.3f' % (d['k1_ms'], d['roofline']['frac'], d['construct_ms']))" || tail -3 gpurun_out/v.err
  done
done
