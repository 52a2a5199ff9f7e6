O=gpurun_out/r02h
mkdir -p $O
ncu --set full --import-source on --clock-control none -k regex:"mr_inv" -c 2 -o $O/c5_k4 python bench.py --config c5 --c5-views 256 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_c5.log 2>&1
tail -1 $O/ncu_c5.log | head -c 200; echo
