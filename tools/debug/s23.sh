timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s23_smoke.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s23_ref.json 2> gpurun_out/s23_ref.err
timeout 600 python bench.py > gpurun_out/s23_bench.json 2> gpurun_out/s23_bench.err
