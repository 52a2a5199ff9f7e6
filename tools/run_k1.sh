python -m pytest tests -m gpu -q -rf > gpurun_out/pytest.log 2>&1; tail -1 gpurun_out/pytest.log
for c in c3 c2 c4; do
for r in 1 4; do
FDL_K1_REPS=$r python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/fb_$c.json 2>gpurun_out/fb_$c.err
python -c "import json;d=json.load(open('gpurun_out/fb_$c.json'));print('$c reps $r', d.get('construct_ms'), d['stages_ms']['k1_ms'], d['roofline']['frac'])"
done
done
