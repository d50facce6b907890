for v in r9b2 r7b2 r7b3 r11b2 r13b2 r5b3 r5b4 r9b3; do
 echo "$v $(DISPCORR_LIB=paper_2508_04951_b200/lib/variants/libdispcorr_$v.so timeout 120 python tools/debug/variant_bench.py 20 256 2>&1 | tail -1)"
done > gpurun_out/s4_dop.log 2>&1
