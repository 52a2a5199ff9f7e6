# repeatability check of the C2 K1 and C5 K3 stage times
O=gpurun_out/recheck
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.mem,clocks.max.sm,power.draw,temperature.gpu --format=csv
for i in 1 2; do
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c2.$i.json 2> $O/c2.$i.err
  python -c "import json;d=json.loads(open('$O/c2.$i.json').read().strip().splitlines()[-1]);print('c2', {k:round(v,3) for k,v in d['stages_ms'].items()})"
  python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5.$i.json 2> $O/c5.$i.err
  python -c "import json;d=json.loads(open('$O/c5.$i.json').read().strip().splitlines()[-1]);print('c5', {k:round(v,3) for k,v in d['stages_ms'].items()})"
done
