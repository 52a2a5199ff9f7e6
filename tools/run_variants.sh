# A/B the prebuilt variants/*.so on the bench (K1 stage time) -- tuning only
for v in variants/*.so; do
  cp $v paper_1901_06919_b200/_lib/libfdl_b200.so
  for c in ${CONFIGS:-c2}; do
    python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/v.json 2>gpurun_out/v.err
    python -c "import json;d=json.load(open('gpurun_out/v.json'));print('$v $c', round(d['construct_ms'],3), {k[:6]:round(x,3) for k,x in d['stages_ms'].items()}, round(d['render']['ms'],3))"
  done
done
