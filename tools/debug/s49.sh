timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/s49_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s49_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s49_bench.json 2> gpurun_out/s49_bench.err
