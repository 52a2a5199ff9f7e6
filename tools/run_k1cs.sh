# K1 CTA-staged spectra A/B (FDL_K1_CTASTAGE) + parity
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py tests/test_gpu_helpers.py -q -x 2>&1 | tail -1
for c in c2 c4 c3 c1; do for cs in 1 0; do
  FDL_K1_CTASTAGE=$cs python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "import json;d=json.load(open('gpurun_out/v.json'));print('$c cs=$cs', 'k1 %.3f frac %.3f construct %.3f' % (d['k1_ms'], d['roofline']['frac'], d['construct_ms']))" || tail -3 gpurun_out/v.err
done; done
