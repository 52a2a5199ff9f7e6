# one ncu --set full capture of the C2 K1 kernel (after a clean run)
O=gpurun_out/k1ncu
mkdir -p $O
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_fast -s 1 -c 1 -o $O/k1_c2 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1; tail -1 $O/ncu.log
