python bench.py --config c3 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('minBlocks2', d['k1_ms'], d['roofline']['frac'])"
sed -i 's/(NB <= 2 ? 3 : (NB <= 6 ? 2 : 1))/(NB <= 2 ? 3 : (NB <= 4 ? 2 : 1))/' paper_1901_06919_b200/csrc/k1_dmma.cu
python paper_1901_06919_b200/build_native.py > /dev/null 2>&1
python bench.py --config c3 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('minBlocks1', d['k1_ms'], d['roofline']['frac'])"
python -m pytest tests/test_gpu_fullsize.py -q -s -k c3 2>&1 | grep -E "rel L2"
