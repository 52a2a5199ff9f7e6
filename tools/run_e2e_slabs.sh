for s in 2 4 8; do
FDL_PIPELINE_SLABS=$s python bench.py --no-cpu-baseline > gpurun_out/b2_$s.json 2>gpurun_out/b2.err; python -c "import json;d=json.load(open('gpurun_out/b2_$s.json'));print('slabs $s', d['construct_ms'], d['e2e']['construct_ms'], d['e2e']['value'])"
done
