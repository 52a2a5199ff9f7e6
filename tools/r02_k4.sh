O=gpurun_out/r02g
mkdir -p $O
python -m pytest tests/test_gpu_fft.py -m gpu -q -x -s -k inverse 2>&1 | grep -E "inv |passed|failed|Error|error" | tail -20
python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
python bench.py --config c5 --c5-views 1024 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
python - <<PY
import json
d=json.loads(open("$O/bench_c5.json").read().strip().splitlines()[-1])
print("c5", d["value"], d.get("stages_ms"), d.get("roofline",{}).get("frac"), d.get("k4_roofline",{}).get("frac"))
PY
