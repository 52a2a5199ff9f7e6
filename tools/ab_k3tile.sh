# K3 aperture tile (C5) after the staging rewrite: parity + C5 bench
O=gpurun_out/k3tile
mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_reference_suite.py -q -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log
python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5.json 2> $O/c5.err
python -c "import json;d=json.loads(open('$O/c5.json').read().strip().splitlines()[-1]);print('c5', d['stages_ms'], 'frac', round(d['roofline']['frac'],3), 'views/s', round(d['value']))"
