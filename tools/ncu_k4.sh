O=gpurun_out/r02j
mkdir -p $O
ncu --set full --import-source on --clock-control none -k regex:"mr_inv" -s 4 -c 2 -o $O/k4 python tools/bench_k4.py 256 > $O/ncu.log 2>&1
tail -2 $O/ncu.log
