# Round measurement sweep: tests, smoke, every config's bench line, the
# reference arm, a launch list and one full ncu capture of the C2 kernels.
O=gpurun_out/sweep
mkdir -p $O
python -m pytest tests -m gpu -q -rf > $O/pytest.log 2>&1; tail -1 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; head -c 200 $O/bench_c2.json; echo
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_c2_reference.json 2> $O/bench_ref.err; head -c 200 $O/bench_c2_reference.json; echo
python bench.py --config calib --steps 10 --warmup 3 > $O/bench_calib.json 2> $O/bench_calib.err; head -c 200 $O/bench_calib.json; echo
python bench.py --impl reference --config calib --steps 2 --warmup 1 > $O/bench_calib_reference.json 2>> $O/bench_calib.err
for c in c1 c2b c3 c4 c5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 > $O/bench_$c.json 2> $O/bench_$c.err; head -c 150 $O/bench_$c.json; echo
done
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k1_fast|fwd_cols|fwd_rows|inv_cols|inv_rows|render_horner2|render_nyquist" -c 6 -o $O/c2_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
tail -1 $O/ncu_full.log
ncu --set full --import-source on --clock-control none -k regex:"calib_" -c 3 -o $O/calib_full python bench.py --config calib --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_calib.log 2>&1
tail -1 $O/ncu_calib.log
