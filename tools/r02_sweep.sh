# Round-2 measurement sweep: tests, smoke, headline bench (C4 + C5) + reference arm, every other config's
# bench line, launch lists of the headline's two halves, K1 DRAM traffic on C4.
O=gpurun_out/r02
mkdir -p $O
python -m pytest tests -m gpu -q -rf > $O/pytest.log 2>&1; tail -2 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py > $O/bench_headline.json 2> $O/bench_headline.err; head -c 300 $O/bench_headline.json; echo
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_ref.err; head -c 200 $O/bench_reference.json; echo
for c in c1 c2 c2b c3 calib; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --steps 10 > $O/bench_$c.json 2> $O/bench_$c.err; head -c 160 $O/bench_$c.json; echo
done
M=gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,dram__bytes_read.sum,dram__bytes_write.sum
F='regex:^(fwd_|inv_|k1_|count_status|symmetrize|sumsq|default_lambda|render_|mr_inv)'
ncu --metrics $M --clock-control none -k "$F" -c 200 --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c4.log 2>&1
ncu --metrics $M --clock-control none -k "$F" -c 200 --csv --log-file $O/launches_c5.csv python bench.py --config c5 --c5-views 512 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c5.log 2>&1
ls -la $O | head -30
