timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fourstep or c2 or compress or roundtrip" > gpurun_out/s14_tests.log 2>&1
timeout 600 python tools/measure_extras.py iono_sweep --out gpurun_out/r1_iono_sweep3.json > gpurun_out/s14.log 2>&1
