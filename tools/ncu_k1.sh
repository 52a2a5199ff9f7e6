O=${O:-gpurun_out/r02k1}
mkdir -p $O
ncu --set full --import-source on --clock-control none -k regex:"k1_fast_kernel" -c 1 -o $O/c4_k1 python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
tail -1 $O/ncu.log | head -c 100; echo
