timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/s16_tests.log 2>&1
timeout 400 python bench.py > gpurun_out/s16_bench.json 2> gpurun_out/s16_bench.err
timeout 300 python tools/debug/taper_bench.py > gpurun_out/s16_taper.log 2>&1
