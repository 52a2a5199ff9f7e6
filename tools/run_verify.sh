O=gpurun_out/verify
mkdir -p $O
python -m pytest tests -m gpu -q -rf -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; cat $O/bench_c2.json; echo
