# K1 A/B: k-step unroll variants (variants/*.so) x bins per warp (FDL_K1_REPS), C2
for v in variants/*.so; do
  cp $v paper_1901_06919_b200/_lib/libfdl_b200.so
  for r in 2 4 8; do
    FDL_K1_REPS=$r python bench.py --config c2 --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/v.json 2>gpurun_out/v.err
    python -c "import json;d=json.load(open('gpurun_out/v.json'));print('$v reps=$r', 'k1 %.3f frac %.3f' % (d['k1_ms'], d['roofline']['frac']))" || tail -3 gpurun_out/v.err
  done
done
cp variants/a_u2.so paper_1901_06919_b200/_lib/libfdl_b200.so
