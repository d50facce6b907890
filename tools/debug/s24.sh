timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/s24_tests.log 2>&1
timeout 600 python tools/measure_extras.py iono_sweep --out gpurun_out/r1b_iono_sweep.json > gpurun_out/s24.log 2>&1
