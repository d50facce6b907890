timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fourstep or largest or correct or compress or roundtrip" > gpurun_out/s19_tests.log 2>&1
timeout 120 python tools/debug/variant_bench.py 20 256 > gpurun_out/s19_bench.log 2>&1
