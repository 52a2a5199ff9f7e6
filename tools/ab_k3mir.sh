# K3 aperture tile with the mirrored shared-memory table (FDL_RENDER_MIRROR): parity + C5 A/B
O=gpurun_out/k3mir
mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_reference_suite.py tests/test_gpu_pipeline.py -q -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for mir in 0 1; do
  FDL_RENDER_MIRROR=$mir python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5.$mir.json 2> $O/c5.$mir.err
  python -c "import json;d=json.loads(open('$O/c5.$mir.json').read().strip().splitlines()[-1]);print('c5 mirror=$mir', d['stages_ms'], 'frac', round(d['roofline']['frac'],3), 'views/s', round(d['value']))"
done
