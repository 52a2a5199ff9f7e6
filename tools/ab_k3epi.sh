# K3 Horner epilogue batching: render parity tests + C2/C3/C4 render stage times
O=gpurun_out/k3epi
mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for cfg in c2 c3 c4; do
  python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/$cfg.json 2> $O/$cfg.err
  python -c "import json;d=json.loads(open('$O/$cfg.json').read().strip().splitlines()[-1]);r=d['render'];print('$cfg', 'k3', round(r['roofline']['k3_ms'],4), 'frac', round(r['roofline']['frac'],3), 'views/s', round(r['value']))"
done
