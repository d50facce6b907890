timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/s12_tests.log 2>&1
timeout 600 python tools/measure_extras.py iono_sweep --out gpurun_out/r1_iono_sweep2.json > gpurun_out/s12.log 2>&1
