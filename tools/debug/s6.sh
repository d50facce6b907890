timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/s6_tests.log 2>&1
timeout 120 python tools/debug/variant_bench.py 20 256 > gpurun_out/s6_bench.log 2>&1
