# K1 mode-2 warps per CTA (FDL_K1_REALA_WARPS variants prebuilt in variants/): C3 K1 stage time
O=gpurun_out/k1reala
mkdir -p $O
cp paper_1901_06919_b200/_lib/libfdl_b200.so $O/default.so.bak
for v in variants/w8.so variants/w6.so variants/w5.so variants/w4.so; do
  cp $v paper_1901_06919_b200/_lib/libfdl_b200.so
  python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 5 > $O/v.json 2> $O/v.err
  python -c "import json;d=json.loads(open('$O/v.json').read().strip().splitlines()[-1]);print('$v', {k:round(x,3) for k,x in d['stages_ms'].items()}, 'frac', round(d['roofline']['frac'],3))"
done
cp variants/w6.so paper_1901_06919_b200/_lib/libfdl_b200.so
python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_reference_suite.py -q -x 2>&1 | tail -1
rm -f $O/default.so.bak
