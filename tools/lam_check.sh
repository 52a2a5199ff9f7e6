# deferred default-lambda read (host prep overlaps K0): GPU tests, smoke, C2 x2 / C3 bench lines
O=gpurun_out/lam
mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; tail -1 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --steps 20 --no-cpu-baseline --no-e2e > $O/bench_c2b_rep.json 2> $O/bench_c2_rep.err
python bench.py --config c3 --steps 5 > $O/bench_c3.json 2> $O/bench_c3.err
for f in bench_c2 bench_c2b_rep bench_c3; do python -c "
import json;d=json.loads([l for l in open('$O/$f.json').read().splitlines() if l.startswith('{')][-1]);r=d['roofline']
print('$f', '%.4g'%d['value'], round(d['construct_ms'],3), {k:round(v,3) for k,v in d.get('stages_ms',{}).items()}, 'frac', round(r['frac'],3), 'stage', round(r.get('frac_stage') or 0,3), 'e2e', d.get('e2e',{}).get('value'))
"; done
