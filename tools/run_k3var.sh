# A/B K3 Horner variants (variants/*.so x FDL_H2_VB): C2 render K3 time
for v in variants/*.so; do
  cp $v paper_1901_06919_b200/_lib/libfdl_b200.so
  for vb in 8 9 10; do
    FDL_H2_VB=$vb python bench.py --config c2 --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/v.json 2>gpurun_out/v.err
    python -c "import json;d=json.load(open('gpurun_out/v.json'));r=d['render'];print('$v vb=$vb', 'k3 %.3f frac %.3f render %.3f' % (r['roofline']['k3_ms'], r['roofline']['frac'], r['ms']))" || tail -3 gpurun_out/v.err
  done
done
cp variants/a_minb4.so paper_1901_06919_b200/_lib/libfdl_b200.so
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_reference_suite.py -q -x 2>&1 | tail -1
