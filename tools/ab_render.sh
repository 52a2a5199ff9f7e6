for vb in 16 8; do
 FDL_RENDER_VB=$vb python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c2 VB', $vb, d['render'])"
 FDL_RENDER_VB=$vb python bench.py --config c5 --steps 2 --warmup 1 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c5 VB', $vb, d['value'], d['render_flops_tf'])"
done
