python -m pytest tests -m gpu -q -rf > gpurun_out/pytest.log 2>&1; tail -3 gpurun_out/pytest.log
for c in c2 c1 c2b c4; do
python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/fb_$c.json 2>gpurun_out/fb_$c.err
python -c "import json;d=json.load(open('gpurun_out/fb_$c.json'));print('$c', d['construct_ms'], d['stages_ms'], d['render'])"
done
