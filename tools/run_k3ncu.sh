# one ncu --set full capture of the C2 K3 Horner tile + C2/C5 render timing
O=gpurun_out/k3ncu
mkdir -p $O
for c in c2 c5; do
python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
python -c "import json; j=json.load(open('$O/bench_$c.json')); r=j['render'] if 'render' in j else j; print('$c', json.dumps(r.get('roofline', j.get('roofline')))[:300], j['stages_ms'] if 'stages_ms' in j else '')"
done
ncu --set full --clock-control none --import-source on -k regex:"render_horner2|render_tile|fwd_rows|fwd_cols|inv_rows|inv_cols" -c 6 -o $O/k3_c2 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1; tail -1 $O/ncu.log
