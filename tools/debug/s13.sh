ncu --set full --import-source on --clock-control none -k regex:"iono_cluster" -s 1 -c 1 -o gpurun_out/s13_prof python tools/debug/iono_driver.py 16 2048 2 > gpurun_out/s13_ncu.log 2>&1
