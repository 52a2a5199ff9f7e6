# source-level ncu capture of K1 on C3 (real-A focal stack path)
O=gpurun_out/k1c3
mkdir -p $O
python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench.log 2>&1 || exit 1
tail -1 $O/bench.log | cut -c1-400
ncu --set full --import-source on --clock-control none -k regex:"k1_fast" -c 1 -o $O/k1 python bench.py --config c3 --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > $O/ncu.log 2>&1
tail -1 $O/ncu.log
