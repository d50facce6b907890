timeout 900 python tools/measure_extras.py all --out gpurun_out/r1b_extras.json > gpurun_out/s54.log 2>&1
timeout 600 python bench.py > gpurun_out/r1b_bench.json 2> gpurun_out/r1b_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1b_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/r1b_launches_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"doppler_pipe|warp_col3_kernel|warp_row_kernel" -s 4 -c 4 -o gpurun_out/r1b_prof python tools/debug/profile_driver.py 20 256 2 > gpurun_out/r1b_prof.log 2>&1
