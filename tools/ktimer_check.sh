# bench lines with the per-launch kernel timer (K1 / K3 roofline over the kernels' own launch durations)
O=gpurun_out/ktimer
mkdir -p $O
python -m pytest tests/test_abi.py tests/test_gpu_helpers.py -q 2>&1 | tail -1
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --config c3 --steps 5 > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --config c5 --no-cpu-baseline --steps 5 > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py --config c4 --no-cpu-baseline --steps 3 > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --config c2b --no-cpu-baseline --steps 5 > $O/bench_c2b.json 2> $O/bench_c2b.err
for c in c2 c3 c5 c4 c2b; do python -c "
import json;d=json.loads([l for l in open('$O/bench_$c.json').read().splitlines() if l.startswith('{')][-1]);r=d['roofline']
print('$c', 'k1' if 'k1_ms' in d else 'k3', round(r['frac'],3), 'stage', round(r.get('frac_stage') or 0,3), 'launch ms', r.get('kernel_ms_per_launch'), r.get('launches_per_step'))
if 'render' in d: rr=d['render']['roofline']; print('   k3', round(rr['frac'],3), 'stage', round(rr['frac_stage'],3), rr.get('kernel_ms_per_launch'), rr.get('launches_per_step'))
"; done
