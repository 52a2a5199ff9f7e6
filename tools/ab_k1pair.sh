# K1 split-system CTA shape (FDL_K1_PAIR_WARPS x FDL_K1_PAIR_MINB variants prebuilt in variants/): C2 K1 stage time
O=gpurun_out/k1pair
mkdir -p $O
for v in variants/p8_3.so variants/p6_4.so variants/p4_6.so variants/p8_4.so variants/p8_3.so; do
  cp $v paper_1901_06919_b200/_lib/libfdl_b200.so
  python bench.py --config c2 --no-cpu-baseline --no-e2e --steps 10 > $O/v.json 2> $O/v.err
  python -c "import json;d=json.loads(open('$O/v.json').read().strip().splitlines()[-1]);print('$v', 'k1', round(d['stages_ms']['k1_ms'],4), 'frac', round(d['roofline']['frac'],4))"
done
