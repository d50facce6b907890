timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/s15_tests.log 2>&1
timeout 120 python tools/debug/variant_bench.py 20 256 > gpurun_out/s15_bench.log 2>&1
