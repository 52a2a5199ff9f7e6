python -m pytest tests -m gpu -q -rf > gpurun_out/pytest.log 2>&1; tail -1 gpurun_out/pytest.log
for c in c2 c3 c4; do
python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/fb_$c.json 2>gpurun_out/fb_$c.err
python -c "import json;d=json.load(open('gpurun_out/fb_$c.json'));print('$c', d.get('construct_ms'), d['stages_ms']['k1_ms'], d['roofline']['frac'])"
done
ncu --set full --import-source on --clock-control none -k regex:"k1_fast" -c 1 -o gpurun_out/k1_c2c python bench.py --config c2 --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > gpurun_out/ncu_k1c2.log 2>&1
