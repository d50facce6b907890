timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "compress" > gpurun_out/s9_tests.log 2>&1
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/s9_all.log 2>&1
