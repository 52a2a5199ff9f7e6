python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest.log 2>&1; tail -1 gpurun_out/pytest.log
python bench.py --no-cpu-baseline > gpurun_out/b2.json 2>gpurun_out/b2.err; python -c "import json;d=json.load(open('gpurun_out/b2.json'));print(d['construct_ms'], d['e2e'])"
