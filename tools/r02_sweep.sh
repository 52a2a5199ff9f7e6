# Round-2 measurement sweep: tests, smoke, headline bench (C4 + C5), reference arm, launch list.
O=gpurun_out/r02a
mkdir -p $O
python -m pytest tests -m gpu -q -rf -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py > $O/bench_headline.json 2> $O/bench_headline.err; head -c 600 $O/bench_headline.json; echo; tail -3 $O/bench_headline.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_ref.err; head -c 300 $O/bench_reference.json; echo
for c in c2 c3; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --steps 10 > $O/bench_$c.json 2> $O/bench_$c.err; head -c 200 $O/bench_$c.json; echo
done
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file $O/launches_headline.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
tail -2 $O/ncu_launch.log
