# after the sizes-only (dry) plans for the path / workspace queries: GPU tests + C3/C5/C2 bench lines
O=gpurun_out/plan
mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; tail -1 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --config c3 --steps 5 > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --config c5 --no-cpu-baseline --steps 5 > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
for c in c3 c5 c2; do python -c "
import json;d=json.loads([l for l in open('$O/bench_$c.json').read().splitlines() if l.startswith('{')][-1]);r=d['roofline']
print('$c', '%.4g'%d['value'], {k:round(v,3) for k,v in d.get('stages_ms',{}).items()}, 'frac', round(r['frac'],3), 'stage', round(r.get('frac_stage') or 0,3), 'e2e', d.get('e2e',{}).get('value'))
"; done
