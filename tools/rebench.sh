# bench lines of C2 (default driver line) and C5, twice each
O=gpurun_out/rebench
mkdir -p $O
for i in 1 2; do
  python bench.py > $O/bench_c2.$i.json 2> $O/bench_c2.$i.err
  timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 5 > $O/bench_c5.$i.json 2> $O/bench_c5.$i.err
done
for f in $O/*.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', d['value'], d.get('stages_ms'), d['roofline']['frac'], d['clocks'])"; done
