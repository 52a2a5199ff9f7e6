# A/B of the pipelined column FFT passes (FDL_FFT_PIPE) on C2, C2b and C4 + FFT parity tests
O=gpurun_out/fftpipe
mkdir -p $O
python -m pytest tests/test_gpu_fft.py tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for cfg in c2 c2b c4; do
  for pipe in 0 1; do
    FDL_FFT_PIPE=$pipe python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/$cfg.$pipe.json 2> $O/$cfg.$pipe.err
    python -c "import json,sys;d=json.loads(open('$O/$cfg.$pipe.json').read().strip().splitlines()[-1]);print('$cfg pipe=$pipe', {k:round(v,3) for k,v in d['stages_ms'].items()}, 'construct', round(d.get('construct_ms',0),3))"
  done
done
