O=gpurun_out/r02e
mkdir -p $O
python -m pytest tests -m gpu -q -x -rf > $O/pytest.log 2>&1; tail -15 $O/pytest.log
python bench.py --config c2 --no-cpu-baseline --steps 10 > $O/bench_c2.json 2> $O/bench_c2.err; python - <<PY
import json
d=json.loads(open("$O/bench_c2.json").read().strip().splitlines()[-1])
print("c2", d["value"], d.get("stages_ms"), d["roofline"]["frac"], d["roofline"].get("kernel_ms_per_launch"))
PY
