python -m pytest tests/test_gpu_fft.py -q -rf -s > gpurun_out/pytest_fft.log 2>&1; tail -30 gpurun_out/pytest_fft.log
grep -E "^fwd|^inv|passed|failed|Error" gpurun_out/pytest_fft.log
