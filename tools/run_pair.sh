# K1 mirror-pair split: parity tests + C2/C4/C1 bench, A/B against FDL_K1_PAIR=0
O=gpurun_out/pair
mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_sharded.py -q -rf -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for c in c2 c4 c1; do
  python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 > $O/bench_$c.json 2> $O/bench_$c.err
  FDL_K1_PAIR=0 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 > $O/bench_${c}_nopair.json 2>> $O/bench_$c.err
  python - <<PY
import json
for f in ["$O/bench_$c.json", "$O/bench_${c}_nopair.json"]:
    try:
        j = json.load(open(f)); print(f, "k1_ms %.3f frac %.3f construct %.3f" % (j["k1_ms"], j["roofline"]["frac"], j["construct_ms"]))
    except Exception as e: print(f, "ERR", e)
PY
done
