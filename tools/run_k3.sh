python -m pytest tests -m gpu -q -rf > gpurun_out/pytest.log 2>&1; tail -1 gpurun_out/pytest.log
for c in c2 c5 c4; do
python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/fb_$c.json 2>gpurun_out/fb_$c.err
python -c "import json;d=json.load(open('gpurun_out/fb_$c.json'));print('$c', d.get('construct_ms'), d.get('stages_ms'), d.get('render'), d.get('value'))"
done
