set -x
mkdir -p /tmp/rep
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:warp_col3|warp_row|doppler_pipe' -s 4 -c 4 -o /tmp/rep/c4full python tools/profile_driver.py 20 256 2 > gpurun_out/f2_ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f2_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/f2_ncu_list.log 2>&1
python tools/profile_summary.py r2d /tmp/rep/c4full.ncu-rep gpurun_out/f2_launches.csv 268435456 > gpurun_out/f2_summary.log 2>&1
python tools/ncu_fp32_ops.py /tmp/rep/c4full.ncu-rep 268435456 > profiles/r2d_fp32_ops.json 2> gpurun_out/f2_fp32.err
cp profiles/r2d_* gpurun_out/ 2>/dev/null
timeout 600 python bench.py > gpurun_out/f2_bench.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f2_gt.log 2>&1; echo rc=$? >> gpurun_out/f2_gt.log
