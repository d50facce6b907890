for v in i2f; do
 echo "$v $(DISPCORR_LIB=paper_2508_04951_b200/lib/variants/libdispcorr_$v.so timeout 120 python tools/debug/variant_bench.py 20 256 2>&1 | tail -1)"
done > gpurun_out/s61.log 2>&1
echo "base $(timeout 120 python tools/debug/variant_bench.py 20 256 2>&1 | tail -1)" >> gpurun_out/s61.log
