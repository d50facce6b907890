ncu --set full --import-source on --clock-control none -k regex:"warp_row_kernel" -s 1 -c 1 -o gpurun_out/s36_prof python tools/debug/iono_driver.py 10 131072 2 > gpurun_out/s36_ncu.log 2>&1
